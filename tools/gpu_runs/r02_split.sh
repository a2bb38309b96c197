# row split kernel: kernel tests, then A/B against the tiles (HL_GATHER_SPLIT=0) on the owner-pack batches
HL_GATHER_SPLIT=1 timeout 900 python -m pytest tests/test_kernel_gpu.py -x -q 2>&1 | tail -2
HL_GATHER_SPLIT=1 compute-sanitizer --tool memcheck python -m pytest tests/test_kernel_gpu.py -x -q -k "row_split" 2>&1 | tail -3
for rep in 1 2; do for S in 0 1; do
  HL_GATHER_SPLIT=$S python tools/kernel_bench.py --variants pack8,cols8 --iters 10 | sed "s/^/split=$S /"
  HL_GATHER_SPLIT=$S python tools/kernel_bench.py --arch llama2-70b --layers 8 --variants pack8,cols8 --iters 10 | sed "s/^/split=$S /"
done; done
