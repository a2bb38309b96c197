# C2 (7B, 13.5 GB warm): engine slot/chunk size x team x slots, DMA-completion timeline
python bench.py --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
for rep in 1 2; do for cfg in "12 3 4194304" "12 2 8388608" "8 2 8388608" "8 3 8388608" "6 2 16777216" "8 2 16777216" "12 3 8388608"; do
  set -- $cfg
  HL_ENGINE_WORKERS=$1 HL_ENGINE_SLOTS=$2 HL_PROBE_BOUNCE=$3 python tools/gpu_runs/c1_timeline.py /tmp/hl_bench/llama2-7b-aligned
done; done
