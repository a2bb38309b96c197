# interleaved tile groups (a tensor's W shards stream the same rows together) vs descriptor-major order
timeout 900 python -m pytest tests/test_kernel_gpu.py tests/test_io_gpu.py -x -q 2>&1 | tail -2
for rep in 1 2; do
for G in 1 16; do
  HL_TILE_GROUP=$G python tools/kernel_bench.py --variants pack8,cols8,pack8cast,cols8cast --iters 10 | sed "s/^/group=$G /"
  HL_TILE_GROUP=$G python tools/kernel_bench.py --arch llama2-70b --layers 8 --variants pack8,cols8,pack8cast,cols8cast --iters 10 | sed "s/^/group=$G /"
done; done
