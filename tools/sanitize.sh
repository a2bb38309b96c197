#!/bin/bash
# compute-sanitizer over hl_gather (race detection / memory checking on the kernel).
# memcheck + initcheck on the kernel and loader tests (the 48 MiB cases excluded: sanitizer replay
# is ~100x slower), racecheck on the kernel tests (the row kernels use warp shuffles; bulk_kernel and staged_kernel stage through shared memory with TMA + mbarriers).
# --show-backtrace device: the sanitizer's host-backtrace capture keeps Python frames (and so the
# loader's views) alive, which trips the loader's own live-view / stale-key checks.
# initcheck --check-api-memory-access no: tests read back whole buffers incl. never-written padding.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
K='--kernel-name kns=row_kernel --kernel-name kns=generic_kernel --kernel-name kns=bulk_kernel --kernel-name kns=staged_kernel'
T=${T:-1500}
for tool in memcheck initcheck racecheck; do
  files="tests/test_kernel_gpu.py"
  [ $tool != racecheck ] && files="$files tests/test_loader_gpu.py tests/test_golden_gpu.py"
  extra="--show-backtrace device"
  [ $tool = initcheck ] && extra="$extra --check-api-memory-access no"
  timeout $T $CS --tool $tool $K $extra --error-exitcode 99 --print-limit 20 --log-file gpurun_out/sanitize_$tool.txt \
      python -m pytest $files -m gpu -q -p no:cacheprovider -k "not large" \
      > gpurun_out/sanitize_${tool}_pytest.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.txt >> gpurun_out/sanitize_summary.txt
  tail -1 gpurun_out/sanitize_${tool}_pytest.log >> gpurun_out/sanitize_summary.txt
done
