# all GPU tests on the current tree + the default bench line
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_4.log 2>&1; tail -3 gpurun_out/r02_gpu_tests_full_4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02_bench_v10.log 2>&1; tail -1 gpurun_out/r02_bench_v10.log > gpurun_out/r02_bench_v10.json
python -c "import json; d=json.load(open('gpurun_out/r02_bench_v10.json')); print(d['value'], d['ms_per_step'], json.dumps(d['e2e_cold']), d['io_roofline']['storage_gbs'], d['io_roofline']['e2e_frac_of_h2d'], json.dumps(d['e2e_fresh_process']), d['roofline']['frac'], d['gpu_launches'], json.dumps(d['clocks']))"
