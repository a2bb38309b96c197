"""HBM held during an auto_release load: allocated bytes after each file's
last key (file buffers should return to the pool then: ref loader.py:501-508)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from bench import ensure_data  # noqa: E402
from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup, synth  # noqa: E402
from paper_2505_23072_b200.format import read_header  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
layers = int(sys.argv[2]) if len(sys.argv) > 2 else None
paths = [str(p) for p in ensure_data(arch, "/tmp/hl_bench", "aligned", 0, 1, None, layers=layers)]
last_key = {}
for p in paths:
    last_key[list(read_header(p).tensors)[-1]] = p
keys = [e[0] for e in synth.entries(arch, layers)]
torch.cuda.synchronize()
torch.cuda.reset_peak_memory_stats()
base = torch.cuda.memory_allocated()
ld = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(auto_release=True))
ld.add_filenames({0: paths})
fb = ld.copy_files_to_device()
rows = [{"after": "copy_files_to_device", "GB": round((torch.cuda.memory_allocated() - base) / 1e9, 2)}]
outs = []
for k in keys:
    outs.append(fb.get_tensor(k))
    if k in last_key:
        row = {"after_last_key_of": Path(last_key[k]).name,
               "GB": round((torch.cuda.memory_allocated() - base) / 1e9, 2)}
        fb._deferred.flush()  # the pending clone batch holds its sources until it launches
        row["GB_after_flush"] = round((torch.cuda.memory_allocated() - base) / 1e9, 2)
        import gc

        gc.collect()
        row["GB_after_gc"] = round((torch.cuda.memory_allocated() - base) / 1e9, 2)
        row["landing_alive"] = sum(1 for hf in fb._hosted.values() if hf.buffer._tensor is not None)
        rows.append(row)
torch.cuda.synchronize()
rows.append({"peak_GB": round((torch.cuda.max_memory_allocated() - base) / 1e9, 2),
             "tensor_GB": round(synth.total_bytes(arch) / 1e9, 2) if layers is None else None})
print(json.dumps(rows))
