python bench.py --quick --cold-steps 0 --steps 1 --warmup 1 > /dev/null 2>&1
for rep in 1 2 3; do for m in default noprep prepfirst; do python tools/gpu_runs/fresh_probe2.py /tmp/hl_bench/llama2-7b-aligned $m; done; done
