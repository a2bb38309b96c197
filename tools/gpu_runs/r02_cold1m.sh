# cold plans on 1 MiB chunks: engine tests, default bench (cold vs storage probe), C1 line, fresh-process probes
timeout 900 python -m pytest tests/test_io_gpu.py tests/test_loader_gpu.py tests/test_configs_gpu.py -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r02_bench_cold1m.log 2>&1; tail -1 gpurun_out/r02_bench_cold1m.log > gpurun_out/r02_bench_cold1m.json
python -c "import json; d=json.load(open('gpurun_out/r02_bench_cold1m.json')); print(d['value'], json.dumps(d['e2e_cold']), d['io_roofline']['storage_gbs'], json.dumps(d['e2e_fresh_process']))"
python bench.py --arch gpt2 --quick --cold-steps 0 --steps 10 --warmup 3 2>/dev/null | tail -1 > gpurun_out/r02_bench_c1_v2.json
python -c "import json; d=json.load(open('gpurun_out/r02_bench_c1_v2.json')); print('C1', d['value'], json.dumps(d['e2e']['phases_ms']))"
for i in 1 2 3; do python tools/gpu_runs/fresh_probe.py /tmp/hl_bench/llama2-7b-aligned; done 2>&1 | tee gpurun_out/r02_fresh_probe.jsonl
