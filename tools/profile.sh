#!/bin/bash
# ncu evidence for hl_gather (one GPU; never wrap a multi-rank command).
#  1) launch list with device times + DRAM bytes (cold-cache, serialised: compare shares)
#  2) one --set full capture per variant of the 7B batch (291 descriptors, 1 launch)
set -x
mkdir -p gpurun_out
V=${VARIANTS:-clone,realign,cast,castodd,f32f16,pack8}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ncu_launches.csv python tools/kernel_bench.py --variants "$V" --iters 1 \
    > gpurun_out/ncu_launches_stdout.log 2>&1
for v in ${FULL:-clone realign castodd}; do
  ncu --set full --clock-control none --import-source on -k regex:"row_kernel|bulk_kernel|staged_kernel" -s 1 -c 1 \
      -o gpurun_out/prof_$v -f python tools/kernel_bench.py --variants $v --iters 1 \
      > gpurun_out/ncu_full_$v.log 2>&1
done
