# staged_kernel empty-barrier release: every consumer thread arrives (new) vs lane 0 after __syncwarp (old)
L=paper_2505_23072_b200/libhbmload.so
cp tools/build/libhbmload_thread.so $L
timeout 900 python -m pytest tests/test_kernel_gpu.py -x -q 2>&1 | tail -1
compute-sanitizer --tool racecheck python -m pytest tests/test_kernel_gpu.py -x -q -k "large_contiguous or long_rows" 2>&1 | tail -2
for rep in 1 2; do for v in thread lane0; do
  cp tools/build/libhbmload_$v.so $L
  python tools/kernel_bench.py --variants realign,cast,castodd,f32f16,f32f16odd,bf16f32 --iters 10 | sed "s/^/$v /"
done; done
cp tools/build/libhbmload_thread.so $L
