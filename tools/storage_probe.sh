#!/bin/bash
# Storage roofline probe on the GPU box: cold O_DIRECT reads at several thread counts / io_uring depths.
mkdir -p gpurun_out
gcc -O2 -pthread -o /tmp/storage_probe tools/storage_probe.c || exit 1
F=/tmp/storage_probe.bin
[ -f $F ] || python - <<'PY'
import numpy as np
rng = np.random.default_rng(0)
with open("/tmp/storage_probe.bin", "wb") as f:
    for _ in range(8):
        f.write(rng.integers(0, 256, size=1 << 30, dtype=np.uint8).tobytes())
PY
sync
/tmp/storage_probe $F > gpurun_out/storage_probe.jsonl 2>&1
rm -f $F
