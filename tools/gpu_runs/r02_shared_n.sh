# the N>1 bench path on the one GPU (ranks share it; gloo stands in for NCCL): both planes, N=2 and N=4
for n in 2 4; do
  HL_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
     --master-port $((29600 + n)) bench.py --gpus $n --steps 2 --warmup 3 --quick --cold-steps 1 > gpurun_out/r02_bench_n${n}_shared_final.log 2>&1
  echo "n=$n rc=$?"; tail -1 gpurun_out/r02_bench_n${n}_shared_final.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], {k: (v['value'], v['retrieve_ms'], v['output_checksums'][:2]) for k, v in d['planes'].items()})"
done
