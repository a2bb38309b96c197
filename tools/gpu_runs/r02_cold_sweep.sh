# cold-team sweep (workers x plan chunk) beside the storage probe on the same box; fresh-process first load split
python bench.py --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1   # generates the 7B files
P=$(ls /tmp/hl_bench/llama2-7b-aligned/*.safetensors)
tools/build/storage_probe $P | tee gpurun_out/r02_cold_sweep_probe.jsonl
for W in 32 48 64; do for C in 1048576 2097152 4194304; do
  HL_COLD_WORKERS=$W HL_PLAN_CHUNK=$C python bench.py --quick --cold-steps 2 --steps 1 --warmup 2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'workers': $W, 'chunk': $C, 'cold': d['e2e_cold']['value'], 's': d['e2e_cold']['seconds_to_ready'], 'resid': d['e2e_cold']['residency_before']}))" | tee -a gpurun_out/r02_cold_sweep.jsonl
done; done
for i in 1 2; do python tools/first_load_probe.py --auto-release --split 2>&1 | tail -4; done | tee gpurun_out/r02_first_load.txt
