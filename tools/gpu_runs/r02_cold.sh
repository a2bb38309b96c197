python -m pytest tests/test_loader_gpu.py tests/test_io_gpu.py -x -q 2>&1 | tail -2
tools/build/hmm_probe /tmp/hl_bench/llama2-7b-aligned/model-00001-of-00002.safetensors 4096 2>&1 | tail -4
python bench.py --steps 3 --warmup 2 --cpu-baseline 0 --cold-steps 2 > gpurun_out/r02_bench_v6.log 2>&1; tail -1 gpurun_out/r02_bench_v6.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['e2e_cold']), json.dumps(d['io_roofline']))"
HL_COLD_WORKERS=12 python bench.py --steps 2 --warmup 2 --quick --cold-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cold12', json.dumps(d['e2e_cold']))"
HL_COLD_WORKERS=48 python bench.py --steps 2 --warmup 2 --quick --cold-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cold48', json.dumps(d['e2e_cold']))"
