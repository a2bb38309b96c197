#!/bin/bash
# ncu evidence for hl_gather (one GPU; never wrap a multi-rank command).
#  1) launch list with device times (cold-cache, serialised: compare shares)
#  2) one --set full capture of the clone batch (291 descriptors, 1 launch)
set -x
mkdir -p gpurun_out
V=${VARIANTS:-clone,realign,cast,pack8}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ncu_launches.csv python tools/kernel_bench.py --variants "$V" --iters 1 \
    > gpurun_out/ncu_launches_stdout.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:row_kernel -s 2 -c 1 \
    -o gpurun_out/prof_clone -f python tools/kernel_bench.py --variants clone --iters 1 \
    > gpurun_out/ncu_full_stdout.log 2>&1
