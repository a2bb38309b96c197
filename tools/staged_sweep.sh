#!/bin/bash
# Tuning sweep of the TMA-staged kernel: builds libhbmload variants with HL_STAGED_* macros
# (here, no GPU needed), then on the box swaps each in and runs tools/kernel_bench.py.
# A variant is KB:STAGES:WARPS:CTAS_PER_SM:ALIGNED_CASTS_TOO:TMA_STORE.
#   build:  bash tools/staged_sweep.sh build      run (gpurun): bash tools/staged_sweep.sh run
set -e
D=paper_2505_23072_b200
V="${VARIANTS:-16:6:16:2:1:0 32:3:16:2:1:0 16:6:24:1:1:0 8:12:16:2:1:0 16:4:8:3:1:0}"
if [ "$1" = build ]; then
  mkdir -p sweep
  for v in $V; do
    IFS=: read kb st w c al ts <<< "$v"
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 -shared -cudart static \
      -DHL_STAGED_IN_KB=$kb -DHL_STAGED_STAGES=$st -DHL_STAGED_WARPS=$w -DHL_STAGED_CTAS=$c -DHL_STAGED_ALIGNED=$al -DHL_STAGED_TMA_STORE=${ts:-0} \
      -o sweep/lib_$v.so $D/csrc/hl_gather.cu $D/csrc/hl_io.cpp $D/csrc/hl_peer.cpp $D/csrc/hl_api.cpp -ldl -lpthread &
  done
  wait
  exit 0
fi
mkdir -p gpurun_out
cp $D/libhbmload.so /tmp/lib_orig.so
for v in $V; do
  cp sweep/lib_$v.so $D/libhbmload.so
  echo "== $v" >> gpurun_out/staged_sweep.log
  [ "${TESTS:-0}" = 1 ] && timeout 300 python -m pytest tests/test_kernel_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1 >> gpurun_out/staged_sweep.log
  timeout 120 python tools/kernel_bench.py --iters 10 --variants ${KV:-cast,castodd,f32f16,realign,f16f32} >> gpurun_out/staged_sweep.log 2>&1
done
cp /tmp/lib_orig.so $D/libhbmload.so
