# fixes + A/Bs: fanout route test, kernel/io tests, tile interleave groups, cold readers (io_uring vs blocking) interleaved
timeout 1500 python -m pytest tests/test_kernel_gpu.py tests/test_io_gpu.py "tests/test_ipc_gpu.py::test_ipc_plane_fanout_route_matches_reference" -x -q 2>&1 | tail -2
bash tools/gpu_runs/r02_tile_group.sh 2>&1 | grep -v "passed\|failed" > gpurun_out/r02_tile_group.jsonl
python bench.py --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
P=$(ls /tmp/hl_bench/llama2-7b-aligned/*.safetensors)
tools/build/storage_probe $P > gpurun_out/r02_ab_probe.jsonl
for rep in 1 2 3 4; do for U in 1 0; do
  HL_COLD_URING=$U python bench.py --quick --cold-steps 2 --steps 1 --warmup 2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['e2e_cold']; print(json.dumps({'rep': $rep, 'uring': $U, 'cold': c['value'], 'modes': c['io_modes'], 'threads': c['io_threads'], 'resid': c['residency_before']}))" | tee -a gpurun_out/r02_cold_ab.jsonl
done; done
tools/build/storage_probe $P >> gpurun_out/r02_ab_probe.jsonl
