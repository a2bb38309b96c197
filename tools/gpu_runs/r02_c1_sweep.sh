# C1 (GPT-2 fp32, 0.5 GB) e2e vs engine chunking / team size
for w in 12 16; do for c in 1048576 2097152 4194304; do
  HL_ENGINE_WORKERS=$w HL_PLAN_CHUNK=$c python bench.py --arch gpt2 --quick --cold-steps 0 --steps 7 --warmup 3 2>/dev/null | grep '^{' | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'workers': $w, 'chunk': $c, 'e2e': d['value'], 'phases': d['e2e']['phases_ms']}))"
done; done
# ncu: launch list of the bench command (value leg + deferred e2e batches), then full captures
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"row_kernel|generic_kernel|bulk_kernel|staged_kernel|tile_" -c 800 --csv \
  --log-file gpurun_out/r02_ncu_launches_bench.csv python bench.py --steps 2 --warmup 3 --quick --cold-steps 0 \
  > gpurun_out/r02_ncu_bench_stdout.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bulk_kernel" -s 2 -c 1 \
  -o gpurun_out/r02_prof_bench_bulk -f python bench.py --steps 1 --warmup 3 --quick --cold-steps 0 > /dev/null 2>&1
for v in cols8 cols8cast pack8 pack8cast; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tile_|bulk_kernel|row_kernel" -s 0 -c 3 \
    -o gpurun_out/r02_prof_$v -f python tools/kernel_bench.py --variants $v --iters 1 > /dev/null 2>&1
done
ls -la gpurun_out/
