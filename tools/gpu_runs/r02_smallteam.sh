timeout 900 python -m pytest tests/test_io_gpu.py -x -q 2>&1 | tail -1
python bench.py --arch gpt2 --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
for i in 1 2; do
python tools/gpu_runs/c1_timeline.py /tmp/hl_bench/gpt2-aligned
HL_SMALL_TEAM=12 python tools/gpu_runs/c1_timeline.py /tmp/hl_bench/gpt2-aligned
done
python bench.py --arch gpt2 --cold-steps 2 --steps 10 --warmup 3 2>/dev/null | tail -1 > gpurun_out/r02_bench_c1_v3.json
python -c "import json; d=json.load(open('gpurun_out/r02_bench_c1_v3.json')); print('C1', d['value'], d['io_roofline']['e2e_frac_of_h2d'], json.dumps(d['e2e']['phases_ms']), json.dumps(d['e2e_cold']))"
