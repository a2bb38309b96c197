#!/bin/bash
# Round-end evidence in one call: full GPU suite (per file), the N=1 bench, the reference arm,
# the ncu launch list of the bench command, and vLLM's weight-loading time with this loader.
mkdir -p gpurun_out
bash tools/gpu_tests.sh > gpurun_out/gpu_tests_summary.log 2>&1
python bench.py > gpurun_out/bench_final.log 2>&1
tail -1 gpurun_out/bench_final.log > gpurun_out/bench_final.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_final.log 2>&1
tail -1 gpurun_out/bench_ref_final.log > gpurun_out/bench_ref_final.json
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"row_kernel|generic_kernel|bulk_kernel|staged_kernel" -c 800 --csv \
    --log-file gpurun_out/ncu_launches_bench.csv python bench.py --steps 2 --warmup 3 --quick --cold 0 \
    > gpurun_out/ncu_bench_stdout.log 2>&1
fi
[ "${VLLM:-1}" = 1 ] && timeout 1500 python tools/vllm_startup.py --runs 2 --modes safetensors,ours \
    > gpurun_out/vllm_startup.jsonl 2> gpurun_out/vllm_startup.err
exit 0
