#!/bin/bash
# Box facts for DESIGN.md: CPU/NUMA/RAM/disk/GPU topology, GDS presence.
set -x
nproc; lscpu | head -30; free -g; df -h / /tmp /dev/shm; mount | grep -E ' / | /tmp ' ; 
nvidia-smi; nvidia-smi topo -m; nvidia-smi -q | grep -i -A3 'PCIe Generation\|Link Width'
ls /proc/driver/nvidia-fs 2>&1; cat /proc/driver/nvidia-fs/stats 2>&1 | head
lsblk -o NAME,SIZE,TYPE,ROTA,MODEL,MOUNTPOINT 2>&1 | head -30
cat /proc/sys/vm/drop_caches 2>&1; echo 3 > /proc/sys/vm/drop_caches && echo DROP_OK
python - <<'PY'
import torch, time, os
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
# pinned H2D bandwidth
n = 1<<30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device='cuda')
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(5): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D pinned GB/s", 5*n/e0.elapsed_time(e1)/1e6)
# misaligned H2D
e0.record();
for _ in range(5): d[993:993+n-4096].copy_(h[7:7+n-4096], non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D pinned misaligned GB/s", 5*(n-4096)/e0.elapsed_time(e1)/1e6)
e0.record();
for _ in range(5): h.copy_(d, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("D2H pinned GB/s", 5*n/e0.elapsed_time(e1)/1e6)
# file write + read
path='/tmp/probe.bin'
t=time.time(); 
with open(path,'wb') as f:
    b = os.urandom(1<<26)
    for _ in range(64): f.write(b)
    f.flush(); os.fsync(f.fileno())
print("write 4GiB GB/s", 4*2**30/(time.time()-t)/1e9)
import numpy as np
buf = np.empty(1<<26, dtype=np.uint8)
fd=os.open(path, os.O_RDONLY)
t=time.time(); off=0
while True:
    k=os.preadv(fd,[buf],off)
    if k<=0: break
    off+=k
print("warm pread 1 thread GB/s", off/(time.time()-t)/1e9)
os.posix_fadvise(fd,0,0,os.POSIX_FADV_DONTNEED)
t=time.time(); off=0
while True:
    k=os.preadv(fd,[buf],off)
    if k<=0: break
    off+=k
print("cold-ish (fadvise) pread 1 thread GB/s", off/(time.time()-t)/1e9)
os.close(fd)
PY
