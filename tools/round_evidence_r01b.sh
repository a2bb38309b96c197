mkdir -p gpurun_out
python bench.py > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"row_kernel|generic_kernel|bulk_kernel" -c 800 --csv --log-file gpurun_out/ncu_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --quick --cold 0 > gpurun_out/ncu_bench_stdout.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_kernel -s 1 -c 1 \
  -o gpurun_out/prof_bench_main -f python bench.py --quick --cold 0 --steps 1 --warmup 3 > gpurun_out/ncu_full_bench.log 2>&1
FULL="clone cast castodd" timeout 1200 bash tools/profile.sh > gpurun_out/profile.log 2>&1
T=900 timeout 2400 bash tools/sanitize.sh > gpurun_out/sanitize.log 2>&1
exit 0
