#!/bin/bash
# Round-end evidence in one call: full GPU suite (per file), the N=1 bench, the reference arm.
mkdir -p gpurun_out
bash tools/gpu_tests.sh > gpurun_out/gpu_tests_summary.log 2>&1
python bench.py > gpurun_out/bench_final.log 2>&1
tail -1 gpurun_out/bench_final.log > gpurun_out/bench_final.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_final.log 2>&1
tail -1 gpurun_out/bench_ref_final.log > gpurun_out/bench_ref_final.json
exit 0
