# refinement: ring footprints <= the 60 MiB L3, two repeats each
python bench.py --arch gpt2 --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
python bench.py --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
for rep in 1 2; do
for D in /tmp/hl_bench/gpt2-aligned /tmp/hl_bench/llama2-7b-aligned; do
for cfg in "6 2 4194304" "4 3 4194304" "5 2 4194304" "4 2 4194304" "8 2 3145728" "6 3 2097152" "12 3 4194304" "7 2 4194304"; do
  set -- $cfg
  HL_ENGINE_WORKERS=$1 HL_ENGINE_SLOTS=$2 HL_PLAN_CHUNK=$3 python tools/gpu_runs/c1_timeline.py $D
done; done; done
