# io_uring cold reader + ipc fanout route: tests, cold bench legs (uring vs blocking readers) beside the storage probe
timeout 1200 python -m pytest tests/test_io_gpu.py tests/test_ipc_gpu.py tests/test_loader_gpu.py -x -q 2>&1 | tail -3
python bench.py --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
P=$(ls /tmp/hl_bench/llama2-7b-aligned/*.safetensors)
tools/build/storage_probe $P > gpurun_out/r02_uring_probe.jsonl; grep io_uring gpurun_out/r02_uring_probe.jsonl | head -3
for rep in 1 2; do
for cfg in "1 2 16" "1 1 32" "1 4 8" "1 2 32" "0 0 0"; do
  set -- $cfg
  HL_COLD_URING=$1 HL_URING_THREADS=$2 HL_URING_DEPTH=$3 python bench.py --quick --cold-steps 2 --steps 1 --warmup 2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'uring': '$1', 'threads': $2, 'depth': $3, 'cold': d['e2e_cold']['value'], 'modes': d['e2e_cold']['io_modes'], 'workers': d['e2e_cold']['io_threads'], 'resid': d['e2e_cold']['residency_before']}))" | tee -a gpurun_out/r02_uring_sweep.jsonl
done; done
