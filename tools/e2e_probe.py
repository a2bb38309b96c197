"""Where does copy_files_to_device spend its time? Same process, same files:
the loader path vs the bare engine (one call for both files / one file)."""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import ensure_data  # noqa: E402
from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup, _native  # noqa: E402


def main():
    paths = ensure_data("llama2-7b", "/tmp/hl_bench", "aligned", 0, 1, None)
    for p in paths:
        Path(p).read_bytes() if os.path.getsize(p) < (1 << 35) else None
    print(json.dumps({"residency": [_native.file_residency(str(p)) for p in paths]}), flush=True)
    for mode in ("auto", "buffered"):
        for i in range(4):
            t0 = time.perf_counter()
            ld = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(io_mode=mode))
            ld.add_filenames({0: [str(p) for p in paths]})
            t1 = time.perf_counter()
            fb = ld.copy_files_to_device()
            t2 = time.perf_counter()
            st = ld.last_transfer_stats
            print(json.dumps({"path": "loader", "mode": mode, "i": i, "add_ms": round((t1 - t0) * 1e3, 2),
                              "copy_ms": round((t2 - t1) * 1e3, 2), "engine_ms": round(st.engine_seconds * 1e3, 2),
                              "read_s": round(st.read_seconds, 3), "wait_s": round(st.wait_seconds, 3),
                              "GBps": round(st.bytes / (t2 - t1) / 1e9, 2), "modes": st.io_modes}), flush=True)
            fb.close()
            ld.close()
    sizes = [os.path.getsize(p) for p in paths]
    dev = [torch.empty(s, dtype=torch.uint8, device="cuda") for s in sizes]
    eng = _native.IoEngine(0, workers=12, chunk_bytes=4 << 20, io_mode="buffered")
    for label, files in (("both", [0, 1]), ("file0", [0]), ("file1", [1])):
        for i in range(3):
            blocks = [(j, 0, 0, sizes[f], dev[f].data_ptr()) for j, f in enumerate(files)]
            st = eng.execute([str(paths[f]) for f in files], blocks)
            print(json.dumps({"path": "engine", "files": label, "i": i, "wall_ms": round(st["seconds"] * 1e3, 2),
                              "GBps": round(st["bytes"] / st["seconds"] / 1e9, 2), "read_s": round(st["read_seconds"], 3),
                              "wait_s": round(st["wait_seconds"], 3), "submit_s": round(st["submit_seconds"], 3)}),
                  flush=True)


if __name__ == "__main__":
    main()
