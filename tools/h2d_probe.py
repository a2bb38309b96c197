"""Pinned H2D bandwidth vs copy size and stream count (the DMA side of the
engine in isolation): 8 GiB per point from a pinned pool into one device
buffer, copies round-robin over S streams."""
import json

import torch

TOTAL = 8 << 30


def run(chunk: int, streams: int) -> float:
    n = TOTAL // chunk
    pool = 48 << 20
    h = torch.empty(pool + chunk, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(TOTAL, dtype=torch.uint8, device="cuda")
    ss = [torch.cuda.Stream() for _ in range(streams)]
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in ss:
            s.wait_event(e0)
        for i in range(n):
            s = ss[i % streams]
            with torch.cuda.stream(s):
                off = (i * chunk) % pool
                d[i * chunk:(i + 1) * chunk].copy_(h[off:off + chunk], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    return TOTAL / (e0.elapsed_time(e1) / 1e3) / 1e9


for chunk_mb in (1, 2, 4, 8, 16, 64):
    for streams in (1, 4, 12):
        print(json.dumps({"chunk_mb": chunk_mb, "streams": streams,
                          "GBps": round(run(chunk_mb << 20, streams), 2)}), flush=True)
