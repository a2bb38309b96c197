# round-2 re-entry: full GPU suite, smoke, default bench, reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full_2.log 2>&1; tail -3 gpurun_out/r02_gpu_tests_full_2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r02_bench_default.log 2>&1; tail -1 gpurun_out/r02_bench_default.log > gpurun_out/r02_bench_default.json; tail -c 600 gpurun_out/r02_bench_default.json
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref.log 2>&1; tail -1 gpurun_out/r02_bench_ref.log > gpurun_out/r02_bench_ref.json; tail -c 400 gpurun_out/r02_bench_ref.json
