python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_full.log 2>&1; tail -3 gpurun_out/r02_gpu_tests_full.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_v4.json 2> gpurun_out/r02_bench_v4.err; tail -c 300 gpurun_out/r02_bench_v4.err
python bench.py --arch gpt2 --quick --cold-steps 1 --steps 5 --warmup 3 > gpurun_out/r02_bench_c1.json 2>&1
