"""Host cost of per-key retrieval: µs per get_tensor (auto-release clone) on the
7B checkpoint, plus a cProfile of one pass (top functions by tottime)."""

from __future__ import annotations

import cProfile
import io
import json
import pstats
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import ensure_data  # noqa: E402
from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup  # noqa: E402
from paper_2505_23072_b200.loader import FilesBufferOnDevice, _HostedFile  # noqa: E402
from paper_2505_23072_b200.device import DeviceBuffer  # noqa: E402


def main():
    paths = ensure_data("llama2-7b", "/tmp/hl_bench", "aligned", 0, 1, None)
    ld = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(auto_release=False))
    ld.add_filenames({0: [str(p) for p in paths]})
    landed = ld.copy_files_to_device()
    keys = list(landed.keys())

    def fresh():
        hosted = {p: _HostedFile(DeviceBuffer(ld.pool, hf.buffer.tensor, hf.buffer.capacity), dict(hf.dev_offsets),
                                 hf.unconsumed) for p, hf in landed._hosted.items()}
        for h in hosted.values():
            h.buffer.refcount = h.unconsumed
        ld.config.auto_release = True
        return FilesBufferOnDevice(ld, hosted)

    res = {}
    for label in ("get_tensor", "get_tensors"):
        times = []
        for i in range(5):
            fb = fresh()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if label == "get_tensor":
                outs = [fb.get_tensor(k) for k in keys]
            else:
                outs = fb.get_tensors(keys)
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            times.append((t1 - t0) * 1e6 / len(keys))
            del outs
            fb._hosted = {}
            fb.close()
        res[label + "_us_per_key"] = round(sorted(times)[2], 2)
    print(json.dumps(res), flush=True)
    for label, fn in (("get_tensor", lambda fb: [fb.get_tensor(k) for k in keys]),
                      ("get_tensors", lambda fb: fb.get_tensors(keys))):
        fb = fresh()
        pr = cProfile.Profile()
        pr.enable()
        outs = fn(fb)
        pr.disable()
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
        print(f"==== {label}\n{s.getvalue()}")
        torch.cuda.synchronize()
        del outs
        fb._hosted = {}
        fb.close()


if __name__ == "__main__":
    main()
