bash tools/gpu_tests.sh > gpurun_out/r02_gpu_tests_summary.log 2>&1; cat gpurun_out/r02_gpu_tests_summary.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench_v5.log 2>&1; tail -1 gpurun_out/r02_bench_v5.log > gpurun_out/r02_bench_v5.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref_v5.log 2>&1; tail -1 gpurun_out/r02_bench_ref_v5.log > gpurun_out/r02_bench_ref_v5.json
