python bench.py --arch gpt2 --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
for rep in 1 2; do for cfg in "6 2097152" "4 2097152" "5 2097152" "6 4194304" "8 2097152" "6 1048576"; do
set -- $cfg
HL_SMALL_TEAM=$1 HL_PLAN_CHUNK=$2 python tools/gpu_runs/c1_timeline.py /tmp/hl_bench/gpt2-aligned
done; done
