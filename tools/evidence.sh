#!/bin/bash
# One gpurun call's worth of round evidence (1 GPU):
#   box facts, reference arm, N=2/N=4 torchrun on the one GPU (HL_SHARE_GPU=1),
#   ncu launch list of the bench command, ncu --set full of the hot kernel variants.
mkdir -p gpurun_out
( nproc; free -g; df -h /tmp ) > gpurun_out/box.txt 2>&1
T=${T:-900}
timeout $T python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
for n in ${SHARED_N:-2 4}; do
  HL_SHARE_GPU=1 timeout $T python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --steps 3 --warmup 3 --quick \
      > gpurun_out/bench_n${n}_shared.log 2>&1
  HL_SHARE_GPU=1 timeout $T python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --impl reference --gpus $n --steps 2 --warmup 1 \
      > gpurun_out/bench_ref_n${n}_shared.log 2>&1
done
# launch list of the bench command itself (cold-cache, serialised: compare shares, not absolutes)
timeout $T ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"row_kernel|generic_kernel|bulk_kernel|staged_kernel" -c 800 --csv --log-file gpurun_out/ncu_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --quick --cold 0 > gpurun_out/ncu_bench_stdout.log 2>&1
[ "${FULL_PROFILE:-1}" = 1 ] && FULL="${FULL:-clone cast castodd}" bash tools/profile.sh > gpurun_out/profile.log 2>&1
exit 0
