"""Sweep the bulk I/O engine: mode x workers x chunk on the bench checkpoint.

  python tools/io_bench.py [--modes buffered,mmap,direct] [--workers 4,8,12,16] [--chunks 4,16,64]

Also measures page-cache -> pinned memory pread bandwidth without any H2D
(how fast the CPU side alone can go) and pinned H2D alone.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2505_23072_b200 import _native  # noqa: E402


def pread_only(path: Path, threads: int, chunk: int) -> float:
    size = path.stat().st_size
    bufs = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(threads)]
    fd = os.open(str(path), os.O_RDONLY)
    cur = [0]
    lock = threading.Lock()

    def work(i):
        mv = memoryview(bufs[i].numpy())
        while True:
            with lock:
                off = cur[0]
                cur[0] += chunk
            if off >= size:
                return
            os.preadv(fd, [mv[: min(chunk, size - off)]], off)

    t0 = time.perf_counter()
    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    os.close(fd)
    return size / dt / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="buffered,mmap,direct")
    ap.add_argument("--workers", default="4,8,12,16")
    ap.add_argument("--chunks", default="4,16,64")
    ap.add_argument("--slots", default="3")
    ap.add_argument("--file", default=None)
    args = ap.parse_args()
    if args.file:
        path = Path(args.file)
    else:
        from bench import ensure_data

        path = ensure_data("llama2-7b", "/tmp/hl_bench", "aligned", 0, 1, None)[0]
    size = path.stat().st_size
    dev = torch.empty(size, dtype=torch.uint8, device="cuda")
    _ = path.read_bytes() if size < (1 << 34) else None  # warm
    if "buffered" in args.modes:
        for t in (4, 8, 12, 16):
            print(json.dumps({"probe": "pread_only_to_pinned", "threads": t, "chunk_mb": 16,
                              "GBps": round(pread_only(path, t, 16 << 20), 2)}), flush=True)
    for mode in args.modes.split(","):
        for w in map(int, args.workers.split(",")):
            for c, sl in [(float(c), int(sl)) for c in args.chunks.split(",") for sl in args.slots.split(",")]:
                eng = _native.IoEngine(0, workers=w, chunk_bytes=int(c * (1 << 20)), slots_per_worker=sl, io_mode=mode)
                res = []
                for i in range(3):
                    if mode == "direct":
                        _native.drop_cache(str(path))
                    st = eng.execute([str(path)], [(0, 0, 0, size, dev.data_ptr())])
                    if i:
                        res.append(size / st["seconds"] / 1e9)
                eng.close()
                print(json.dumps({"mode": mode, "workers": w, "chunk_mb": c, "slots": sl, "GBps": round(max(res), 2),
                                  "modes_used": st["io_modes"], "ring_setup_s": round(st["ring_setup_seconds"], 4),
                                  "read_s": round(st["read_seconds"], 3), "wait_s": round(st["wait_seconds"], 3),
                                  "submit_s": round(st["submit_seconds"], 3), "wall_s": round(st["seconds"], 3)}),
                      flush=True)
                if mode == "direct" and w >= 8 and c >= 16:
                    break


if __name__ == "__main__":
    main()
