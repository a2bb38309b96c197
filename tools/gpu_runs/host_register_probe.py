"""Can this host pin page-cache pages of a file mapping for DMA
(cudaHostRegister on an mmap of the file)? Prints one line per flag set."""
import ctypes as C
import mmap
import os

import numpy as np
import torch

torch.cuda.init()
rt = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if rt is None:
    import glob
    rt = C.CDLL(glob.glob("/usr/local/cuda*/lib64/libcudart.so*")[0])
rt.cudaHostRegister.argtypes = [C.c_void_p, C.c_size_t, C.c_uint]
rt.cudaHostUnregister.argtypes = [C.c_void_p]
rt.cudaGetErrorString.restype = C.c_char_p
libc = C.CDLL(None)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
p = "/tmp/hr_probe.bin"
open(p, "wb").write(np.random.default_rng(0).integers(0, 256, 8 << 20, dtype=np.uint8).tobytes())
open(p, "rb").read()
fd = os.open(p, os.O_RDONLY)
fdrw = os.open(p, os.O_RDWR)
PROT_READ, PROT_WRITE, MAP_SHARED, MAP_PRIVATE, MAP_POPULATE = 1, 2, 1, 2, 0x8000
attr = C.c_int()
rt.cudaDeviceGetAttribute.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_int]
rt.cudaDeviceGetAttribute(C.byref(attr), 113, 0)  # cudaDevAttrHostRegisterReadOnlySupported
print("HostRegisterReadOnlySupported", attr.value)
print("kernel", os.uname().release)
for name, prot, flags, f in [("shared-ro", PROT_READ, MAP_SHARED, fd), ("shared-ro-populate", PROT_READ, MAP_SHARED | MAP_POPULATE, fd),
                             ("shared-rw", PROT_READ | PROT_WRITE, MAP_SHARED, fdrw)]:
    for rflags, rname in [(0x1 | 0x8, "portable|readonly"), (0x1, "portable"), (0x0, "default")]:
        a = libc.mmap(None, 8 << 20, prot, flags, f, 0)
        e = rt.cudaHostRegister(a, 8 << 20, rflags)
        print(name, rname, e, rt.cudaGetErrorString(e).decode())
        if e == 0:
            rt.cudaHostUnregister(a)
        rt.cudaGetLastError()
