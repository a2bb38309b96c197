"""Where does a per-key get_tensor spend host time? cProfile over the
retrieval loop of a warm load (C1 gpt2 and C2 llama2-7b)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import ensure_data, warm_cache  # noqa: E402
from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup  # noqa: E402

arch = sys.argv[1] if len(sys.argv) > 1 else "gpt2"
paths = [str(p) for p in ensure_data(arch, "/tmp/hl_bench", "aligned", 0, 1, None)]
warm_cache(paths)
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ld = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(auto_release=True))
    ld.add_filenames({0: paths})
    fb = ld.copy_files_to_device()
    t1 = time.perf_counter()
    keys = fb.keys()
    if i == 3:
        pr = cProfile.Profile()
        pr.enable()
    outs = [fb.get_tensor(k) for k in keys]
    if i == 3:
        pr.disable()
    t2 = time.perf_counter()
    outs[-1].torch.reshape(-1)[:8].cpu()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{arch} load {1e3*(t1-t0):.2f} ms, retrieve enqueue {1e3*(t2-t1):.2f} ms for {len(keys)} keys "
          f"({1e6*(t2-t1)/len(keys):.1f} us/key), drain {1e3*(t3-t2):.2f} ms, engine {1e3*ld.last_transfer_stats.engine_seconds:.2f} ms")
    del outs
    fb.close()
    ld.close()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
