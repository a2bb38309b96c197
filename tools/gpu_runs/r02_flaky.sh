# flakiness check: the driver's GPU suite twice more, then three bench lines on one box
for i in 1 2; do timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02_flaky_$i.log 2>&1; tail -1 gpurun_out/r02_flaky_$i.log; done
for i in 1 2 3; do timeout 900 python bench.py --cold-steps 1 --cpu-baseline 0 2>/dev/null | tail -1 > gpurun_out/r02_bench_rep$i.json
python -c "import json; d=json.load(open('gpurun_out/r02_bench_rep$i.json')); print(d['value'], d['io_roofline']['h2d_gbs'], d['e2e_cold']['value'], d['io_roofline']['storage_gbs'], d['roofline']['frac'])"; done
