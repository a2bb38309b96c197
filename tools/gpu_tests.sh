#!/bin/bash
# Run every test file's GPU tests separately under its own timeout; logs per file.
# (pytest exit 5 = the file has no gpu-marked tests.)
mkdir -p gpurun_out
rc=0
for f in tests/test_*.py; do
  n=$(basename "$f" .py)
  timeout "${PER_FILE_TIMEOUT:-600}" python -m pytest "$f" -m gpu -q --timeout 240 --timeout-method=thread \
      -p no:cacheprovider > "gpurun_out/$n.log" 2>&1
  e=$?
  [ $e -eq 5 ] && continue
  echo "EXIT $e" >> "gpurun_out/$n.log"
  echo "$n: $(tail -2 gpurun_out/$n.log | head -1) (exit $e)"
  [ $e -ne 0 ] && rc=1
done
exit $rc
