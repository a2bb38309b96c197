# final ncu evidence: launch list of the bench command (device times + DRAM bytes; cold-cache, serialised:
# compare shares), one --set full capture of the dominant kernel (the value leg's batched bulk copy) and
# of the TP=8 owner-pack tile kernels (interleave groups)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02f_launches.csv python bench.py --quick --cold-steps 0 --steps 2 --warmup 1 \
    > gpurun_out/r02f_launches_stdout.log 2>&1; echo "launch list rc $?"
ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 1 -c 1 \
    -o gpurun_out/r02f_bulk -f python tools/kernel_bench.py --variants clone --iters 1 > gpurun_out/r02f_bulk.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"tile_copy_kernel|tile_cast_kernel" -s 0 -c 2 \
    -o gpurun_out/r02f_tiles -f python tools/kernel_bench.py --variants cols8,cols8cast --iters 1 > gpurun_out/r02f_tiles.log 2>&1
ls -la gpurun_out/*.ncu-rep
for i in 1 2 3; do python tools/gpu_runs/fresh_probe.py /tmp/hl_bench/llama2-7b-aligned 2>&1 | head -1; done > gpurun_out/r02f_fresh.jsonl
