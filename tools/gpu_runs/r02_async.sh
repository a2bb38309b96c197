python -m pytest tests/test_io_gpu.py tests/test_loader_gpu.py tests/test_ipc_gpu.py tests/test_configs_gpu.py tests/test_acceptance_gpu.py tests/test_golden_gpu.py -x -q 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_v7.log 2>&1; tail -1 gpurun_out/r02_bench_v7.log > gpurun_out/r02_bench_v7.json
python -c "import json; d=json.load(open('gpurun_out/r02_bench_v7.json')); print(d['value'], json.dumps(d['e2e']['phases_ms']), json.dumps(d['e2e_cold']), d['io_roofline']['storage_gbs'], d['io_roofline']['h2d_gbs'], d['e2e_fresh_process'])"
python bench.py --arch gpt2 --quick --cold-steps 0 --steps 7 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1', d['value'], json.dumps(d['e2e']['phases_ms']))"
