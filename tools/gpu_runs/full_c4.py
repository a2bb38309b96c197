"""C4 at full size on one B200: the whole Llama-2-70B checkpoint (137.95 GB of
bf16 tensors, 15 files, HF split) from a warm page cache (files on the box's
tmpfs: /dev/shm has 197 GB, the disk 67 GB free) through the drop-in API with
the reference default auto_release=True: get_tensor every key, every file
buffer released as its last key is consumed, so HBM peaks near the checkpoint
plus one file (179 GiB card). Prints one JSON line: load GB/s, seconds to
ready, peak HBM, engine phases, and a bit-exact check of sampled tensors
against the files."""
import json
import os
import random
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from bench import ensure_data  # noqa: E402
from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup, synth  # noqa: E402
from paper_2505_23072_b200.format import read_header  # noqa: E402

data_dir = sys.argv[1] if len(sys.argv) > 1 else "/dev/shm/hl_full"
t0 = time.time()
paths = [str(p) for p in ensure_data("llama2-70b", data_dir, "aligned", 0, 1, None)]
gen_s = time.time() - t0
keys = [e[0] for e in synth.entries("llama2-70b")]
tensor_bytes = synth.total_bytes("llama2-70b")
where = {}
for p in paths:
    h = read_header(p)
    for k, m in h.tensors.items():
        where[k] = (p, h.body_offset + m.begin, m.nbytes)
rows = []
for it in range(4):
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    t = time.perf_counter()
    ld = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(auto_release=True))
    ld.add_filenames({0: paths})
    fb = ld.copy_files_to_device()
    t1 = time.perf_counter()
    outs = [fb.get_tensor(k) for k in keys]
    t2 = time.perf_counter()
    tail = outs[-1].torch.reshape(-1)[:32].view(torch.uint8).cpu()
    torch.cuda.synchronize()
    s = time.perf_counter() - t
    st = ld.last_transfer_stats
    ms = torch.cuda.memory_stats()
    row = {"iter": it, "seconds_to_ready": round(s, 3), "GBps": round(tensor_bytes / s / 1e9, 2),
           "copy_s": round(t1 - t, 3), "retrieve_s": round(t2 - t1, 3), "drain_s": round(s - (t2 - t), 3),
           "engine_s": round(st.engine_seconds, 3), "io_modes": st.io_modes, "io_threads": st.io_threads,
           "peak_allocated_GB": round(ms.get("allocated_bytes.all.peak", 0) / 1e9, 1),
           "peak_reserved_GB": round(ms.get("reserved_bytes.all.peak", 0) / 1e9, 1),
           "alloc_retries": ms.get("num_alloc_retries"), "cuda_malloc_retries": ms.get("num_device_alloc")}
    if it == 3:  # bit-exact against the file bytes, 24 sampled tensors (the largest included)
        rng = random.Random(7)
        sample = rng.sample(keys, 23) + [max(keys, key=lambda k: where[k][2])]
        ok = True
        for k in sample:
            p, off, nb = where[k]
            ref = np.fromfile(p, dtype=np.uint8, count=nb, offset=off)
            ok &= outs[keys.index(k)].tobytes() == ref.tobytes()
        row["sampled_bit_exact"] = {"tensors": len(sample), "ok": bool(ok)}
    rows.append(row)
    del outs, tail
    fb.close()
    ld.close()
    torch.cuda.empty_cache()
med = sorted(r["seconds_to_ready"] for r in rows[1:])[1]
print(json.dumps({"workload": "llama2-70b bf16 synthetic, full 80 blocks, 15 files (HF split), N=1, get_tensor every key, "
                                "auto_release=True, files on tmpfs (warm)",
                  "tensor_bytes": tensor_bytes, "files": len(paths), "generate_s": round(gen_s, 1),
                  "value_GBps": round(tensor_bytes / med / 1e9, 2), "seconds_to_ready": med, "iters": rows}))
