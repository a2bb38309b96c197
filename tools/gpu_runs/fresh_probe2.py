"""First load of a fresh process, split: what does the kernel-preparation side
thread cost, and the first carve chunk? argv[2] = default | noprep | prepfirst."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

torch.empty(1, device="cuda:0")
from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup, _native  # noqa: E402

mode = sys.argv[2]
out = {"mode": mode}
if mode == "noprep":
    _native._prepared.add(0)  # no side thread: kernels load lazily at their first launch
elif mode == "prepfirst":
    t = time.perf_counter()
    _native.gather_prepare(0)
    out["prepare_ms"] = round((time.perf_counter() - t) * 1e3, 2)
paths = sorted(str(p) for p in Path(sys.argv[1]).glob("*.safetensors"))
t0 = time.perf_counter()
ld = SafeTensorsFileLoader(SingleGroup(), "cuda:0", config=LoaderConfig(auto_release=True))
ld.add_filenames({0: paths})
fb = ld.copy_files_to_device()
t1 = time.perf_counter()
keys = fb.keys()
a = time.perf_counter()
first = fb.get_tensor(keys[0])
t_first = time.perf_counter() - a
outs = [first] + [fb.get_tensor(k) for k in keys[1:]]
t2 = time.perf_counter()
torch.cuda.synchronize()
t3 = time.perf_counter()
st = ld.last_transfer_stats
out.update({"copy_ms": round((t1 - t0) * 1e3, 2), "engine_ms": round(st.engine_seconds * 1e3, 2),
            "ring_setup_ms": round(st.ring_setup_seconds * 1e3, 2), "first_get_ms": round(t_first * 1e3, 2),
            "retrieve_ms": round((t2 - t1) * 1e3, 2), "sync_ms": round((t3 - t2) * 1e3, 2),
            "total_ms": round((t3 - t0) * 1e3, 2)})
print(json.dumps(out), flush=True)
