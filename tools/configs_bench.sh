#!/bin/bash
# bench.py on every BASELINE.json config that one B200 box can hold (1 GPU, ~80 GB free disk):
#   C1 GPT-2 fp32 (aligned; odd header on the GDS-shaped landing = realign kernel; f32->f16 cast)
#   C2 Llama-2-7B bf16 (the headline config)
#   C3 Llama-2-13B bf16 full at N=1, then TP=2 / TP=4 get_sharded as torchrun ranks sharing the GPU
#   C4 Llama-2-70B bf16, first 24 blocks (disk), N=1
#   C5 Bloom-176B bf16, first 8 blocks (disk), on-device fp16 cast; cold leg included
mkdir -p gpurun_out
D=${HL_BENCH_DIR:-/tmp/hl_bench}
T=${T:-1500}
run() { local name=$1; shift; timeout $T "$@" > gpurun_out/cfg_$name.log 2>&1; echo "$name exit $?"; }
run c1 python bench.py --arch gpt2 --steps 5 --warmup 3
run c1_odd_gds python bench.py --arch gpt2 --header odd --backend gds --steps 5 --warmup 3
run c1_f16 python bench.py --arch gpt2 --cast F16 --steps 5 --warmup 3
rm -rf $D/gpt2-*
run c2 python bench.py --steps 5 --warmup 3
rm -rf $D/llama2-7b-*
run c3 python bench.py --arch llama2-13b --steps 3 --warmup 3
for n in 2 4; do
  HL_SHARE_GPU=1 run c3_tp$n python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py --arch llama2-13b --gpus $n --steps 3 --warmup 3 --quick --data-plane ipc
done
rm -rf $D/llama2-13b-*
run c4_l24 python bench.py --arch llama2-70b --layers 24 --steps 3 --warmup 3
# C4 shape at TP=8 (8 ranks sharing the GPU): both data planes (NCCL plane = gloo-staged here)
HL_SHARE_GPU=1 run c4_l4_tp8 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
    --master-port 29718 bench.py --arch llama2-70b --layers 4 --gpus 8 --steps 2 --warmup 2 --quick --cold-steps 1
rm -rf $D/llama2-70b-*
run c5_l8_f16 python bench.py --arch bloom-176b --layers 8 --cast F16 --steps 3 --warmup 3
HL_SHARE_GPU=1 run c5_l2_tp8_f16 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
    --master-port 29728 bench.py --arch bloom-176b --layers 2 --cast F16 --gpus 8 --steps 2 --warmup 2 --quick --cold-steps 1
rm -rf $D/bloom-176b-*
df -h /tmp > gpurun_out/cfg_df.txt
exit 0
