# split kernel width threshold: tiles only (0) vs split up to 1 / 2 / 4 KiB / every width
for rep in 1 2; do for M in 0 1024 2048 4096 1073741824; do
  if [ $M = 0 ]; then E="HL_GATHER_SPLIT=0"; else E="HL_SPLIT_MAX_SEG=$M"; fi
  env $E python tools/kernel_bench.py --variants pack8,cols8,pack8cast --iters 10 | sed "s/^/maxseg=$M /"
  env $E python tools/kernel_bench.py --arch llama2-70b --layers 8 --variants pack8,cols8 --iters 10 | sed "s/^/maxseg=$M /"
done; done
