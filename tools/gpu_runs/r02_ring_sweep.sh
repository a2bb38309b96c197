# ring footprint vs the 60 MiB L3 (DMA reads of recently written slots): workers x slots x chunk, C1 and C2, DMA-completion timeline
python bench.py --arch gpt2 --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
python bench.py --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
for D in /tmp/hl_bench/gpt2-aligned /tmp/hl_bench/llama2-7b-aligned; do
for W in 6 8 12; do for S in 2 3; do for C in 2097152 4194304; do
  HL_ENGINE_WORKERS=$W HL_ENGINE_SLOTS=$S HL_PLAN_CHUNK=$C python tools/gpu_runs/c1_timeline.py $D
done; done; done; done
