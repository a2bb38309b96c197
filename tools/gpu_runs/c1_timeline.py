"""Timeline of one small warm load (C1 GPT-2 0.5 GB): host phase times and
GPU event times (all relative to the start), to split the e2e into
header parse / engine submission / DMA completion / retrieval / drain."""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup  # noqa: E402

paths = sorted(str(p) for p in Path(sys.argv[1]).glob("*.safetensors"))
nbytes = sum(os.path.getsize(p) for p in paths)
rows = []
for i in range(12):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    ev[0].record()
    bounce = int(os.environ.get("HL_PROBE_BOUNCE", "0"))  # engine slot size (LoaderConfig.host_bounce_bytes)
    cfg = LoaderConfig(auto_release=True, **({"host_bounce_bytes": bounce} if bounce else {}))
    ld = SafeTensorsFileLoader(SingleGroup(), "cuda:0", config=cfg)
    ld.add_filenames({0: paths})
    t1 = time.perf_counter()
    fb = ld.copy_files_to_device()
    t2 = time.perf_counter()
    ev[1].record()
    outs = [fb.get_tensor(k) for k in fb.keys()]
    t3 = time.perf_counter()
    ev[2].record()
    tail = outs[-1].torch.reshape(-1)[:32].view(torch.uint8).cpu()
    ev[3].record()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    st = ld.last_transfer_stats
    g = [ev[0].elapsed_time(e) for e in ev[1:]]
    rows.append({"add": (t1 - t0) * 1e3, "copy_ret": (t2 - t0) * 1e3, "engine": st.engine_seconds * 1e3,
                 "last_submit": (t1 - t0) * 1e3 + st.last_h2d_seconds * 1e3,
                 "gpu_dma_done": g[0], "retr_ret": (t3 - t0) * 1e3, "gpu_retr_done": g[1], "gpu_tail_done": g[2],
                 "wall": (t4 - t0) * 1e3})
    del outs, tail
    fb.close()
    ld.close()
rows = rows[3:]
med = {k: round(sorted(r[k] for r in rows)[len(rows) // 2], 3) for k in rows[0]}
med["GBps_wall"] = round(nbytes / med["wall"] / 1e6, 2)
med["GBps_dma"] = round(nbytes / (med["gpu_dma_done"] - med["add"]) / 1e6, 2)
med["env"] = {k: v for k, v in os.environ.items() if k.startswith("HL_")}
print(json.dumps(med), flush=True)
