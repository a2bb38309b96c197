"""Golden API-semantics traces from the REFERENCE loader (build container only;
the reference does not exist on the GPU box). Re-run:
    python tests/golden/make_ops_golden.py   -> tests/golden/ops_cases.json

Each scenario takes one of the committed golden corpora (tests/golden/corpora),
a world size (thread ranks of one ProcessGroup), a backend and auto_release,
and drives the reference's SafeTensorsFileLoader with a random op sequence
that every rank issues in the same order:

  ("tensor", key) / ("shard", key, dim)  -> get_tensor / get_sharded
  ("drop", i)                            -> forget op i's result (+ gc): survivors die
  ("close",)                             -> FilesBufferOnDevice.close()
  ("read", i)                            -> tobytes() of op i's result after the fact

Repeated keys (live buffer, surviving view, stale), unknown keys, bad dims,
use after close and auto-release all appear. Per rank and op the outcome is
["ok", shape, sha256] or ["err", ClassName]; tests/test_ops_gpu.py replays the
same sequences on the B200 loader and demands identical outcomes.
"""

from __future__ import annotations

import gc
import hashlib
import json
import sys
import threading
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

from aggload.collective import ProcessGroup  # noqa: E402  (reference code, read-only import)
from aggload.format import read_header  # noqa: E402
from aggload.loader import LoaderConfig, SafeTensorsFileLoader  # noqa: E402
from aggload.transfer import NumaNode, Topology  # noqa: E402


def make_ops(rng, keys, shapes, n):
    ops = []
    for _ in range(n):
        r = rng.random()
        k = keys[int(rng.integers(0, len(keys)))] if rng.random() > 0.05 else "no_such_key"
        if r < 0.45:
            ops.append(["tensor", k])
        elif r < 0.8:
            rank = len(shapes.get(k, ()))
            ops.append(["shard", k, int(rng.integers(-1, rank + 1)) if rng.random() < 0.15 else int(rng.integers(0, max(rank, 1)))])
        elif r < 0.92 and ops:
            ops.append(["drop", int(rng.integers(0, len(ops)))])
        elif ops:
            ops.append(["read", int(rng.integers(0, len(ops)))])
    if rng.random() < 0.5:
        at = int(rng.integers(len(ops) // 2, len(ops) + 1))
        ops.insert(at, ["close"])
        ops.append(["read", int(rng.integers(0, at))] if at else ["close"])
        ops.append(["tensor", keys[0]])
    return ops


def run(files, world, backend, auto, ops):
    mapping = {r: [str(p) for i, p in enumerate(files) if i % world == r] for r in range(world)}
    topo = Topology((NumaNode(0, 32, tuple(range(world)), (0,)),))
    group = ProcessGroup(world, timeout=20)
    out = [None] * world

    def rank_main(rank):
        ld = SafeTensorsFileLoader(group, rank=rank, config=LoaderConfig(backend=backend, topology=topo,
                                                                         auto_release=auto))
        ld.add_filenames(mapping)
        fb = ld.copy_files_to_device()
        held, trace = {}, []
        for i, op in enumerate(ops):
            try:
                if op[0] == "tensor":
                    v = fb.get_tensor(op[1])
                    held[i] = v
                    trace.append(["ok", list(v.shape), hashlib.sha256(v.tobytes()).hexdigest()])
                elif op[0] == "shard":
                    v = fb.get_sharded(op[1], op[2])
                    held[i] = v
                    trace.append(["ok", list(v.shape), hashlib.sha256(v.tobytes()).hexdigest()])
                elif op[0] == "drop":
                    held.pop(op[1], None)
                    gc.collect()
                    trace.append(["ok"])
                elif op[0] == "read":
                    v = held.get(op[1])
                    trace.append(["ok", hashlib.sha256(v.tobytes()).hexdigest()] if v is not None else ["ok"])
                elif op[0] == "close":
                    fb.close()
                    trace.append(["ok"])
            except Exception as e:  # noqa: BLE001 - the class name is the outcome
                trace.append(["err", type(e).__name__])
        out[rank] = trace
        fb.close()
        ld.close()

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
    return out


def main():
    corpora = json.loads((HERE / "corpora" / "expect.json").read_text())["cases"]
    rng = np.random.default_rng(0x0B5)
    cases = []
    for ci in range(100):
        c = corpora[int(rng.integers(0, len(corpora)))]
        files = [HERE / "corpora" / f for f in c["files"]]
        world = int(rng.integers(1, 5))
        backend = ["host", "simdirect"][int(rng.integers(0, 2))]
        auto = bool(rng.integers(0, 2))
        shapes = {}
        for p in files:
            for k, m in read_header(p).tensors.items():
                shapes[k] = tuple(m.shape)
        keys = sorted(shapes)
        ops = make_ops(rng, keys, shapes, int(rng.integers(8, 50)))
        traces = run(files, world, backend, auto, ops)
        if any(t is None for t in traces):
            continue  # a rank hung (never expected); skip rather than record garbage
        cases.append({"files": [f.name for f in files], "world": world, "backend": backend, "auto_release": auto,
                      "ops": ops, "ranks": traces})
    (HERE / "ops_cases.json").write_text(json.dumps({"cases": cases}) + "\n")
    errs = sum(1 for c in cases for t in c["ranks"] for o in t if o[0] == "err")
    print(f"wrote {len(cases)} scenarios, {sum(len(c['ops']) for c in cases)} ops, {errs} error outcomes")


if __name__ == "__main__":
    main()
