"""Calibrate the reference arm: the oracle PORT of the reference's CPU pipeline
(what bench.py --impl reference times on the GPU box, where the Python
reference cannot travel) against the REFERENCE ITSELF, on the same files in
this build container. Same workload shape as the bench: get_tensor every key
(get_sharded along the Megatron dims at W>1), auto_release=True (the
reference default), warm page cache, W thread-ranks.

    python tools/calibrate_port.py [--gb 2] [--world 1,2]

Prints one JSON line per world size with both GB/s; run here, not on the box.
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(1, "/root/reference/pkg/src")  # reference code, read-only import (build container only)


def make_corpus(d: Path, gb: float):
    from paper_2505_23072_b200 import synth

    layers = max(1, int(gb * 1e9 / 405e6))  # a llama2-7b block is ~405 MB
    return synth.generate("llama2-7b", d, layers=layers, max_bytes=int(gb * 1e9 / 2) + 1)


def time_reference(paths, world, policy):
    from aggload.collective import ProcessGroup
    from aggload.loader import LoaderConfig, SafeTensorsFileLoader

    group = ProcessGroup(world)
    mapping = {r: [str(p) for i, p in enumerate(paths) if i % world == r] for r in range(world)}
    ready = [0] * world

    def rank_main(r):
        ld = SafeTensorsFileLoader(group, rank=r, config=LoaderConfig(backend="host", auto_release=True))
        ld.add_filenames(mapping)
        fb = ld.copy_files_to_device()
        nb = 0
        for k in fb.keys():
            d = policy.get(k) if world > 1 else None
            v = fb.get_tensor(k) if d is None else fb.get_sharded(k, d)
            nb += v.nbytes
        ready[r] = nb
        fb.close()
        ld.close()

    t0 = time.perf_counter()
    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return sum(ready), time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gb", type=float, default=2.0)
    ap.add_argument("--world", default="1,2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dir", default="/tmp/hl_calib")
    args = ap.parse_args()
    import bench
    from paper_2505_23072_b200 import synth

    d = Path(args.dir)
    paths = sorted(d.glob("*.safetensors")) or make_corpus(d, args.gb)
    policy = {n: synth.shard_dim(n, s) for n, _, s in synth.entries("llama2-7b")}
    bench.warm_cache(paths)
    for world in map(int, args.world.split(",")):
        ref, port = [], []
        for _ in range(args.reps):
            nb, t = time_reference(paths, world, policy)
            ref.append(nb / t / 1e9)
            port.append(bench.run_cpu_reference(paths, steps=1, warmup=0, world=world, policy=policy)["value"])
        print(json.dumps({"world": world, "files": len(paths), "ready_bytes": nb,
                          "reference_GBps": round(statistics.median(ref), 3),
                          "port_GBps": round(statistics.median(port), 3),
                          "port_over_reference": round(statistics.median(port) / statistics.median(ref), 3)}),
              flush=True)


if __name__ == "__main__":
    main()
