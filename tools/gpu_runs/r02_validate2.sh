# final-tree validation: full GPU suite, smoke, default bench, reference arm, C1 odd/gds line
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_6.log 2>&1; tail -3 gpurun_out/r02_gpu_tests_full_6.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02_bench_v13.log 2>&1; tail -1 gpurun_out/r02_bench_v13.log > gpurun_out/r02_bench_v13.json
python -c "import json; d=json.load(open('gpurun_out/r02_bench_v13.json')); print(d['value'], d['ms_per_step'], json.dumps(d['e2e_cold']), d['io_roofline']['storage_gbs'], d['io_roofline']['e2e_frac_of_h2d'], json.dumps(d['e2e_fresh_process']), d['roofline']['frac'], d['gpu_launches'], json.dumps(d['clocks']))"
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref_v6.log 2>&1; tail -1 gpurun_out/r02_bench_ref_v6.log > gpurun_out/r02_bench_ref_v6.json; tail -c 200 gpurun_out/r02_bench_ref_v6.json
timeout 900 python bench.py --arch gpt2 --header odd --backend gds --steps 5 --warmup 3 2>/dev/null | tail -1 > gpurun_out/r02_c1_odd_gds_v3.json
python -c "import json; d=json.load(open('gpurun_out/r02_c1_odd_gds_v3.json')); print('C1 odd gds', d['value'], json.dumps(d['e2e']['phases_ms']))"
