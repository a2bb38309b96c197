"""Fresh-process first load (bench.py's e2e_fresh_process leg) with per-phase
and per-call timers: where does a new process's first load spend its time?"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

torch.empty(1, device="cuda:0")
from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup  # noqa: E402

paths = sorted(str(p) for p in Path(sys.argv[1]).glob("*.safetensors"))
for load in range(2):
    t0 = time.perf_counter()
    ld = SafeTensorsFileLoader(SingleGroup(), "cuda:0", config=LoaderConfig(auto_release=True))
    ld.add_filenames({0: paths})
    t1 = time.perf_counter()
    fb = ld.copy_files_to_device()
    t2 = time.perf_counter()
    calls = []
    outs = []
    for k in fb.keys():
        a = time.perf_counter()
        outs.append(fb.get_tensor(k))
        calls.append((time.perf_counter() - a, k))
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    st = ld.last_transfer_stats
    calls.sort(reverse=True)
    print(json.dumps({"load": load, "add_ms": round((t1 - t0) * 1e3, 2), "copy_ms": round((t2 - t1) * 1e3, 2),
                      "engine_ms": round(st.engine_seconds * 1e3, 2), "ring_setup_ms": round(st.ring_setup_seconds * 1e3, 2),
                      "engine_setup_ms": round(st.setup_seconds * 1e3, 2),
                      "first_h2d_ms": round(st.first_h2d_seconds * 1e3, 2),
                      "retrieve_ms": round((t3 - t2) * 1e3, 2), "sync_ms": round((t4 - t3) * 1e3, 2),
                      "total_ms": round((t4 - t0) * 1e3, 2),
                      "slowest_calls": [(round(s * 1e3, 2), k) for s, k in calls[:6]]}), flush=True)
    del outs
    fb.close()
    ld.close()
