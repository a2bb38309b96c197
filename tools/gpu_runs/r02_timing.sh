timeout 900 python -m pytest tests/test_kernel_gpu.py tests/test_abi.py tests/test_smoke_gpu.py -x -q 2>&1 | tail -1
python bench.py --quick --cold-steps 0 --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C2', d['value'], r['achieved'], r['frac'], r['achieved_all_launches_of_step'], r['kernel_share_of_step'])"
python bench.py --arch gpt2 --quick --cold-steps 0 --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C1', d['value'], r['achieved'], r['frac'], r['achieved_all_launches_of_step'], r['kernel_share_of_step'])"
python bench.py --arch gpt2 --cast F16 --quick --cold-steps 0 --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C1 f16', d['value'], r['achieved'], r['frac'], r['kernel'])"
python tools/kernel_bench.py --variants clone,cast,pack8 --iters 10
