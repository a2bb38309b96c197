python -m pytest tests/test_kernel_gpu.py -x -q 2>&1 | tail -3
for t in 1 0; do HL_GATHER_TILES=$t python tools/kernel_bench.py --variants pack8,cols8,pack8cast,cols8cast --iters 5 | sed "s/^/tiles=$t /"; done
for t in 1 0; do HL_GATHER_TILES=$t python tools/kernel_bench.py --arch llama2-70b --layers 8 --variants pack8,cols8,pack8cast,cols8cast --iters 5 | sed "s/^/tiles=$t /"; done
