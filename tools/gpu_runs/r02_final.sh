# final validation of the round-2 tree: driver's GPU suite, smoke, default bench, reference arm, C1 (+f16) lines
rm -rf /tmp/hl_bench /dev/shm/hl_full; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpu_tests_final4.log 2>&1; tail -1 gpurun_out/r02_gpu_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
sleep 20; cat /proc/loadavg
timeout 900 python bench.py > gpurun_out/r02_bench_final3.log 2>&1; tail -1 gpurun_out/r02_bench_final3.log > gpurun_out/r02_bench_final3.json
python -c "import json; d=json.load(open('gpurun_out/r02_bench_final3.json')); print(d['value'], d['ms_per_step'], d['io_roofline']['e2e_frac_of_h2d'], json.dumps(d['e2e_cold']), d['io_roofline']['storage_gbs'], d['io_roofline'].get('cold_frac_of_storage'), json.dumps(d['e2e_fresh_process']), d['roofline']['frac'], d['gpu_launches'], json.dumps(d['clocks']))"
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref_final3.log 2>&1; tail -1 gpurun_out/r02_bench_ref_final3.log > gpurun_out/r02_bench_ref_final3.json
python -c "import json; d=json.load(open('gpurun_out/r02_bench_ref_final3.json')); print('ref', d['value'], d['cpu_baseline']['kind'], json.dumps(d['e2e_cold']))"
for a in "--arch gpt2" "--arch gpt2 --cast F16"; do python bench.py $a --cold-steps 1 --steps 10 --warmup 3 --cpu-baseline 0 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', d['value'], d['io_roofline']['e2e_frac_of_h2d'], d['roofline']['frac'], json.dumps(d['e2e']['phases_ms']))"; done
