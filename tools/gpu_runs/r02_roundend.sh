# the driver's round-end sequence on the current tree: full GPU suite, smoke, default bench, reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_3.log 2>&1; tail -3 gpurun_out/r02_gpu_tests_full_3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r02_bench_final.log 2>&1; tail -1 gpurun_out/r02_bench_final.log > gpurun_out/r02_bench_final.json
python -c "import json; d=json.load(open('gpurun_out/r02_bench_final.json')); print(d['value'], d['ms_per_step'], json.dumps(d['e2e_cold']), d['io_roofline']['storage_gbs'], d['io_roofline']['e2e_frac_of_h2d'], json.dumps(d['e2e_fresh_process']), d['roofline']['frac'], json.dumps(d['cpu_baseline'].get('naive_sequential')))"
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref_final.log 2>&1; tail -1 gpurun_out/r02_bench_ref_final.log > gpurun_out/r02_bench_ref_final.json; tail -c 300 gpurun_out/r02_bench_ref_final.json
