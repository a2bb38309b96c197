"""Golden outcomes of the REFERENCE's shard partitioning (collective.partition,
collective.py:28-74) over random shapes x dims x world sizes, including the
BadDim / DimTooSmall rejections (build container only).
Re-run:  python tests/golden/make_partition_golden.py  -> partition_cases.json
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

from aggload.collective import partition  # noqa: E402  (reference code, read-only import)
from aggload.format import DType, TensorMetadata  # noqa: E402


def main():
    rng = np.random.default_rng(7)
    cases = []
    for _ in range(400):
        rank = int(rng.integers(0, 4))
        shape = [int(x) for x in rng.integers(0, 40, size=rank)]
        dim = int(rng.integers(-1, rank + 2))
        world = int(rng.integers(1, 10))
        n = int(np.prod(shape, dtype=np.int64)) if shape else 1
        meta = TensorMetadata(name="k", dtype=DType.BF16, shape=tuple(shape), data_offsets=(0, 2 * n))
        try:
            spec = partition(meta, dim, world)
            out = {"part_shapes": [list(p) for p in spec.part_shapes], "bounds": [list(spec.bounds(r)) for r in range(world)]}
        except Exception as e:  # noqa: BLE001
            out = {"error": type(e).__name__}
        cases.append({"shape": shape, "dim": dim, "world": world, "expect": out})
    (HERE / "partition_cases.json").write_text(json.dumps({"cases": cases}) + "\n")
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
