set -x
python -m pytest tests/test_io_gpu.py -x -q > gpurun_out/r02_io_tests.log 2>&1; tail -2 gpurun_out/r02_io_tests.log
for pin in 1 0 1 0; do HL_PIN_PAGE_CACHE=$pin python bench.py --quick --cold-steps 0 --steps 5 --warmup 2 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pin=$pin', d['value'], d['e2e']['phases_ms'], d['e2e']['io_modes'])" >> gpurun_out/r02_pin_ab.txt; done
cat gpurun_out/r02_pin_ab.txt
python bench.py --steps 3 --warmup 2 > gpurun_out/r02_bench_v3.json 2> gpurun_out/r02_bench_v3.err; tail -c 400 gpurun_out/r02_bench_v3.err
HL_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --quick --cold-steps 1 --steps 2 --warmup 1 > gpurun_out/r02_bench_n2_shared.json 2> gpurun_out/r02_bench_n2_shared.err; tail -c 1500 gpurun_out/r02_bench_n2_shared.err
