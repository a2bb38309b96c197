import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2505_23072_b200 import _native
p = "/tmp/pin_blob.bin"
data = np.random.default_rng(1).integers(0, 256, 64 << 20, dtype=np.uint8)
open(p, "wb").write(data.tobytes())
open(p, "rb").read()
print("residency", _native.file_residency(p))
dst = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
for mode, flags in (("mmap", 0), ("auto", 1)):
    eng = _native.IoEngine(0, workers=2, chunk_bytes=4 << 20, io_mode=mode, flags=flags)
    print(mode, flags, eng.config)
    st = eng.execute([p], [(0, 0, 0, 64 << 20, dst.data_ptr())], after_stream=0)
    print(mode, st["io_modes"], st["mmap_bytes"], st["buffered_bytes"])
    assert np.array_equal(dst.cpu().numpy(), data)
