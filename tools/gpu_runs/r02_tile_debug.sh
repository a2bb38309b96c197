python tools/gpu_runs/host_register_probe.py 2>&1 | tail -12
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_kernel_gpu.py -x -q -k "test_column_shard_tiles and 0-1-1" 2>&1 | grep -v "^$" | head -60
