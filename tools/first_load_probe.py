"""Cost of the FIRST load in a fresh process (what a model server pays once):
phase times of load 1 vs load 2 of the 7B checkpoint, warm page cache."""
import json
import sys
import time
from pathlib import Path

t_start = time.perf_counter()
import torch  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import ensure_data, warm_cache  # noqa: E402

paths = [str(p) for p in ensure_data("llama2-7b", "/tmp/hl_bench", "aligned", 0, 1, None)]
warm_cache(paths)
t0 = time.perf_counter()
torch.cuda.init()
torch.empty(1, device="cuda")
t_cuda = time.perf_counter() - t0
from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup  # noqa: E402

if "--split" in sys.argv:  # attribute the first load's fixed costs
    from paper_2505_23072_b200 import _native, transfer

    t0 = time.perf_counter()
    x = torch.empty(13_500_000_000, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    del x
    eng = transfer.engine_for(0, transfer.engine_team(), 4 << 20, "auto")
    t2 = time.perf_counter()
    print(json.dumps({"cuda_malloc_13_5GB_ms": round((t1 - t0) * 1e3, 1),
                      "engine_create_ms": round((t2 - t1) * 1e3, 1)}), flush=True)

AUTO = "--auto-release" in sys.argv  # per-key clones (the reference default) instead of views
for i in range(3):
    t0 = time.perf_counter()
    ld = SafeTensorsFileLoader(SingleGroup(), "cuda:0", config=LoaderConfig(auto_release=AUTO))
    ld.add_filenames({0: paths})
    t1 = time.perf_counter()
    fb = ld.copy_files_to_device()
    t2 = time.perf_counter()
    ts = [fb.get_tensor(k).torch for k in fb.keys()]
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    st = ld.last_transfer_stats
    print(json.dumps({"load": i, "add_ms": round((t1 - t0) * 1e3, 1), "copy_ms": round((t2 - t1) * 1e3, 1),
                      "engine_ms": round(st.engine_seconds * 1e3, 1), "ring_setup_ms": round(st.ring_setup_seconds * 1e3, 1),
                      "views_ms": round((t3 - t2) * 1e3, 1), "total_ms": round((t3 - t0) * 1e3, 1),
                      "cuda_init_ms": round(t_cuda * 1e3, 1) if i == 0 else None}), flush=True)
    del ts
    fb.close()
    ld.close()
