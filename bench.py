"""Benchmark: model load GB/s and seconds to ready device tensors on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Workload (BASELINE.json configs[1]): synthetic Llama-2-7B bf16, 2 safetensors
files (13,476,831,232 tensor bytes, 291 tensors, HF order/split, values
N(0,0.02) rounded to bf16), 1 x B200, get_tensor for every key with the
reference's default auto_release=True. The files are generated on the box
(GPU RNG, written once to --data-dir) before anything is timed.
At N > 1 the same checkpoint is loaded tensor-parallel: files round-robin to
ranks, get_sharded with Megatron dims over NCCL, norms replicated
(strong scaling: the model is fixed as N grows).

One JSON line on rank 0:
  value  — HBM-resident leg: file bytes already landed in HBM, one step makes
           every tensor ready (auto-release clones through the batched
           get_tensors, one hl_gather launch) — tensor GB/s, CUDA events.
  e2e    — the drop-in API end to end from files on disk (page cache warm):
           SafeTensorsFileLoader.add_filenames -> copy_files_to_device ->
           get_tensor per key -> synchronize + a D2H read of a result checksum.
           "e2e_cold" repeats it after dropping the page cache.
  roofline   — hl_gather: algorithmic bytes (read+write) / launch time vs the
               measured HBM copy peak (MEASURED_PEAKS.json).
  io_roofline — measured storage read (O_DIRECT, warm pread) and pinned H2D.
  cpu_baseline — the reference's CPU pipeline (oracle port) on a bounded
               sample, on this box's host cores.
--impl reference: that CPU pipeline is the measured arm (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "model load GB/s & seconds to ready device tensors"
SHARE_GPU = os.environ.get("HL_SHARE_GPU") == "1"  # exercise the N>1 code path on a 1-GPU box
ARCH = "llama2-7b"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--arch", default=ARCH)
    ap.add_argument("--header", default="aligned", choices=["aligned", "odd"])
    ap.add_argument("--backend", default="host")
    ap.add_argument("--data-dir", default=os.environ.get("HL_BENCH_DIR", "/tmp/hl_bench"))
    ap.add_argument("--cold", type=int, default=1, help="also time e2e after dropping the page cache")
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--quick", action="store_true", help="skip io probes, cpu and library baselines")
    ap.add_argument("--baselines", type=int, default=1,
                    help="also time upstream fastsafetensors and safetensors on the same files (N=1)")
    ap.add_argument("--files", type=int, default=0,
                    help="re-split the checkpoint into this many files (0: HF split at N=1, N files at N>1)")
    ap.add_argument("--layers", type=int, default=None,
                    help="keep only the first N transformer blocks (configs larger than one GPU / the disk)")
    ap.add_argument("--cast", default=None, help="on-device dtype conversion at retrieval, e.g. F16 (C5)")
    ap.add_argument("--data-plane", default="auto", choices=["auto", "ipc", "nccl"],
                    help="N>1: peer-memory pulls (one hl_gather per rank over NVLink) or NCCL broadcast/scatter")
    return ap.parse_args()


# ----------------------------------------------------------------------------- data
def ensure_data(arch: str, data_dir: str, header: str, rank: int, world: int, dist, files: int | None = None,
                layers: int | None = None):
    """Generate the synthetic checkpoint once per box (GPU RNG). ``files``
    re-splits it HF-style into that many roughly equal files (same tensors,
    same order) so that at N ranks every rank owns file bytes to read."""
    from paper_2505_23072_b200 import synth

    ents = synth.entries(arch, layers)
    max_bytes = None
    if files:
        # greedy split: shrink the cap until the file count is reached (or cannot shrink further)
        cap = -(-sum(synth.nbytes(e) for e in ents) // files)
        while len(synth.split_files(arch, ents, cap)) > files:
            cap = int(cap * 1.02) + 1
        max_bytes = cap
    tag = f"{arch}-{header}" + (f"-L{layers}" if layers is not None else "") + (f"-f{files}" if max_bytes else "")
    d = Path(data_dir) / tag
    marker = d / "READY"
    if rank == 0 and not marker.exists():
        import shutil

        import torch

        need = int(sum(synth.nbytes(e) for e in ents) * 1.05) + (1 << 30)
        Path(data_dir).mkdir(parents=True, exist_ok=True)
        if shutil.disk_usage(data_dir).free < need:
            # make room: drop OUR other generated checkpoints (READY-marked dirs next to this one)
            for other in sorted(Path(data_dir).iterdir()):
                if other != d and (other / "READY").exists():
                    shutil.rmtree(other, ignore_errors=True)
                    if shutil.disk_usage(data_dir).free >= need:
                        break
        t0 = time.time()
        synth.generate(arch, d, header=header, seed=0, device="cuda" if torch.cuda.is_available() else None,
                       max_bytes=max_bytes, layers=layers)
        os.sync()
        marker.write_text(json.dumps({"seconds": time.time() - t0}))
    if world > 1:
        dist.barrier()
    groups = synth.split_files(arch, ents, max_bytes)
    return [d / f"model-{i + 1:05d}-of-{len(groups):05d}.safetensors" for i in range(len(groups))]


def synth_split(arch, layers=None):
    from paper_2505_23072_b200 import synth

    return synth.split_files(arch, synth.entries(arch, layers))


def warm_cache(paths, threads: int = 16, chunk: int = 64 << 20) -> None:
    """Pull the files back into the page cache with buffered reads (the
    engine's O_DIRECT reads of a cold file do not populate it)."""
    import threading

    work = [(str(p), off) for p in paths for off in range(0, os.path.getsize(p), chunk)]
    lock = threading.Lock()

    def run():
        while True:
            with lock:
                if not work:
                    return
                path, off = work.pop()
            fd = os.open(path, os.O_RDONLY)
            try:
                os.pread(fd, chunk, off)
            finally:
                os.close(fd)

    ts = [threading.Thread(target=run) for _ in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()


def residency(paths) -> float:
    """Byte-weighted page-cache residency of the files (mincore)."""
    from paper_2505_23072_b200 import _native

    sizes = [os.path.getsize(p) for p in paths]
    return round(sum(_native.file_residency(str(p)) * n for p, n in zip(paths, sizes)) / max(sum(sizes), 1), 4)


def host_memory() -> dict:
    """MemTotal / MemAvailable / Cached in GB (/proc/meminfo)."""
    out = {}
    try:
        for line in open("/proc/meminfo"):
            k, v = line.split(":")
            if k in ("MemTotal", "MemAvailable", "Cached"):
                out[k] = round(int(v.split()[0]) / 1e6, 1)
    except OSError:
        pass
    return out


def drop_cache(paths):
    from paper_2505_23072_b200 import _native

    for p in paths:
        _native.drop_cache(str(p))
    try:  # system-wide drop when permitted (root on the box)
        with open("/proc/sys/vm/drop_caches", "w") as f:
            f.write("1\n")
    except OSError:
        pass


# ----------------------------------------------------------------------------- clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/hl_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        self.path.unlink(missing_ok=True)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU legs
def run_cpu_reference(paths, steps: int, warmup: int, world: int = 1, policy=None, cast=None):
    """The reference's CPU load pipeline (oracle port of aggload's loader) on
    the FULL workload of this arm: W thread-ranks (the reference's in-process
    ProcessGroup), files round-robin to ranks, each rank's thread-rule preadv
    workers land its files (transfer.py:197-201, 305-389), then every rank
    retrieves every key — an auto-release clone (loader.py:456-461) or its
    slice along the Megatron dim (collective.py:318-330) — from the owner's
    host buffer. ``cast``: the reference's loader cannot convert (SURVEY
    §8a a7), so its conversion (device.convert_dtype = numpy astype) is applied
    to each retrieved tensor. Returns ready tensor bytes per second over all ranks."""
    import threading

    from oracle import oracle

    mapping = {r: [p for i, p in enumerate(paths) if i % world == r] for r in range(world)}
    workers = {r: oracle.thread_rule(len(mapping[r])) for r in range(world)}
    policy = policy or {}
    times, ready = [], 0
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        loaders = {r: oracle.CpuLoader(mapping[r], workers=workers[r]) for r in range(world) if mapping[r]}
        ts = [threading.Thread(target=ld.copy) for ld in loaders.values()]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        owner = {k: ld for ld in loaders.values() for k in ld.index}
        got = [0] * world
        # the reference's broadcast / scatter rendezvous twice per key (the data
        # exchange and the "done" exchange, collective.py:175-255)
        meet = threading.Barrier(world) if world > 1 else None

        def retrieve(r):
            nb = 0
            for k, ld in owner.items():
                d = policy.get(k) if world > 1 else None
                tag = cast.value if cast is not None else None
                if meet:
                    meet.wait()
                nb += (ld.get_tensor(k, tag) if d is None else ld.get_sharded(k, d, world, r, tag)).nbytes
                if meet:
                    meet.wait()
            got[r] = nb

        ts = [threading.Thread(target=retrieve, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        dt = time.perf_counter() - t0
        del loaders, owner
        ready = sum(got)
        if i >= warmup:
            times.append(dt)
    t = statistics.median(times)
    threads = max(sum(workers.values()), world)
    return {"value": ready / t / 1e9, "unit": "GB/s", "cores": threads, "kind": "port", "seconds": t,
            "sample": f"full workload: {len(paths)} file(s), {ready} ready tensor bytes over {world} rank(s), warm "
                      f"page cache; reference thread rule per rank ({sorted(set(workers.values()))} preadv "
                      f"worker(s)), then {world} retrieval thread(s) meeting twice per key (auto-release clones"
                      + (" / Megatron-dim slices" if world > 1 else "")
                      + (f", numpy {cast.value} conversion" if cast is not None else "")
                      + f"); host os.cpu_count()={os.cpu_count()}"}


# ----------------------------------------------------------------------------- io probes
def io_probes(paths, device_index: int):
    """Measured I/O roofline terms: pinned H2D, warm buffered read, cold O_DIRECT read."""
    import torch

    from paper_2505_23072_b200 import _native

    out = {}
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device_index}")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    out["h2d_gbs"] = 4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
    del h, d
    big = paths[0]
    size = os.path.getsize(big)
    dev = torch.empty(size, dtype=torch.uint8, device=f"cuda:{device_index}")
    for mode in ("buffered", "direct"):
        eng = _native.IoEngine(device_index, io_mode=mode)
        if mode == "direct":
            _native.drop_cache(str(big))
        st = eng.execute([str(big)], [(0, 0, 0, size, dev.data_ptr())])
        if mode == "buffered":  # second pass: fully warm
            st = eng.execute([str(big)], [(0, 0, 0, size, dev.data_ptr())])
        out[f"{mode}_read_to_hbm_gbs"] = size / st["seconds"] / 1e9
        eng.close()
    del dev
    # storage-only read rate (no GPU in the loop): O_DIRECT, 16 threads
    _native.drop_cache(str(big))
    out["storage_direct_read_gbs"] = _storage_read(big)
    return out


def _storage_read(path, threads: int = 16, chunk: int = 16 << 20) -> float:
    import mmap
    import threading

    size = os.path.getsize(path)
    fd = os.open(str(path), os.O_RDONLY | os.O_DIRECT)
    cursor = [0]
    lock = threading.Lock()

    def work():
        buf = mmap.mmap(-1, chunk)
        while True:
            with lock:
                off = cursor[0]
                cursor[0] += chunk
            if off >= size:
                break
            os.preadv(fd, [buf], off)
        buf.close()

    t0 = time.perf_counter()
    ts = [threading.Thread(target=work) for _ in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    os.close(fd)
    return size / dt / 1e9


def library_baselines(paths, device_index: int, tensor_bytes: int, steps: int = 3) -> dict:
    """Same files, same box, warm page cache, every key ready on the GPU
    (median of ``steps`` after one warm-up): the paper's own implementation
    (upstream fastsafetensors 0.3.1 from the image, GDS off since the box has
    no nvidia-fs: its pread + bounce-buffer path; get_tensor returns views)
    and the paper's baseline (safetensors ``load_file(device="cuda")``)."""
    import torch

    dev = f"cuda:{device_index}"
    out = {}

    def timed(fn, n):
        ts = []
        for i in range(n + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            if i:
                ts.append(time.perf_counter() - t0)
        return statistics.median(ts)

    try:
        import fastsafetensors
        from fastsafetensors import SafeTensorsFileLoader as FstLoader

        def fst():
            ld = FstLoader(None, dev, nogds=True)
            ld.add_filenames({0: [str(p) for p in paths]})
            fb = ld.copy_files_to_device()
            ts = [fb.get_tensor(k) for k in ld.get_keys()]
            torch.cuda.synchronize()
            del ts
            fb.close()
            ld.close()

        t = timed(fst, steps)
        out["fastsafetensors"] = {"version": getattr(fastsafetensors, "__version__", "0.3.1"), "mode": "nogds",
                                  "value": round(tensor_bytes / t / 1e9, 3), "unit": "GB/s", "seconds": round(t, 4)}
    except Exception as e:  # noqa: BLE001 - a baseline that cannot run is reported, not fatal
        out["fastsafetensors"] = {"error": f"{type(e).__name__}: {e}"[:200]}
    try:
        import safetensors
        from safetensors.torch import load_file

        def st():
            ts = [load_file(str(p), device=dev) for p in paths]
            torch.cuda.synchronize()
            del ts

        t = timed(st, max(1, steps - 1))
        out["safetensors"] = {"version": safetensors.__version__, "call": "load_file(device=cuda)",
                              "value": round(tensor_bytes / t / 1e9, 3), "unit": "GB/s", "seconds": round(t, 4)}
    except Exception as e:  # noqa: BLE001
        out["safetensors"] = {"error": f"{type(e).__name__}: {e}"[:200]}
    return out


FRESH = r"""
import json, sys, time
sys.path.insert(0, {root!r})
import torch
torch.empty(1, device="cuda:{dev}")  # CUDA context first: not part of the load
from paper_2505_23072_b200 import LoaderConfig, SafeTensorsFileLoader, SingleGroup
t0 = time.perf_counter()
ld = SafeTensorsFileLoader(SingleGroup(), "cuda:{dev}", config=LoaderConfig(backend={backend!r}, auto_release=True))
ld.add_filenames({{0: {paths!r}}})
fb = ld.copy_files_to_device()
outs = [fb.get_tensor(k) for k in fb.keys()]
torch.cuda.synchronize()
print(json.dumps({{"seconds": time.perf_counter() - t0}}))
"""


def e2e_fresh_process(paths, device_index: int, backend: str, job_bytes: int) -> dict | None:
    """The same e2e load as the FIRST load of a fresh process (what a model
    server pays once: engine threads, pinned ring, allocator growth, kernel
    module loading), CUDA context creation excluded; warm page cache."""
    code = FRESH.format(root=str(ROOT), dev=device_index, backend=backend, paths=[str(p) for p in paths])
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
        secs = json.loads(r.stdout.strip().splitlines()[-1])["seconds"]
    except Exception as e:  # noqa: BLE001 - reported, not fatal
        return {"error": f"{type(e).__name__}: {e}"[:200]}
    return {"value": round(job_bytes / secs / 1e9, 3), "unit": "GB/s", "seconds_to_ready": round(secs, 4),
            "note": "first load in a new process (CUDA context excluded), auto_release=True, warm page cache"}


def hbm_peak_gbs() -> tuple[float, str]:
    """Roofline denominator: the driver-measured copy bandwidth, else the
    fallback B200_PROFILING.md states (6.65 TB/s, an earlier measurement)."""
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(peaks["hbm_gbs"]), "of measured: MEASURED_PEAKS.json hbm_gbs (burst copy)"
    except (OSError, ValueError, KeyError, TypeError):
        return 6650.0, "of fallback: B200_PROFILING.md 6.65 TB/s (MEASURED_PEAKS.json absent)"


# ----------------------------------------------------------------------------- GPU legs
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist

    if world > 1:
        if SHARE_GPU:  # test mode: every rank on cuda:0, gloo control plane (NCCL refuses shared GPUs)
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # at N ranks every rank must own file bytes: re-split only when the HF split has fewer than N files
    hf_files = len(synth_split(args.arch, args.layers))
    n_files = args.files if args.files else (None if world <= hf_files else world)
    paths = ensure_data(args.arch, args.data_dir, args.header, rank, world, dist, n_files, args.layers)
    from paper_2505_23072_b200 import synth

    from paper_2505_23072_b200.format import DType

    ents = synth.entries(args.arch, args.layers)
    tensor_bytes = sum(synth.nbytes(e) for e in ents)
    cast = DType.from_tag(args.cast.upper()) if args.cast else None
    src_dt = ents[0][1]
    dtype_tag = src_dt.value.lower() + (f"->{cast.value.lower()}" if cast else "")
    workload = (f"{args.arch}{f' (first {args.layers} blocks)' if args.layers is not None else ''} "
                f"{src_dt.value.lower()} synthetic, {len(paths)} files, "
                + ("get_tensor every key" if world == 1 else f"TP={world} get_sharded (Megatron dims)")
                + (f", on-device {src_dt.value}->{cast.value} cast" if cast else ""))
    file_bytes = sum(os.path.getsize(p) for p in paths)

    if args.impl == "reference":
        if rank == 0:
            policy = {e[0]: synth.shard_dim(e[0], e[2]) for e in ents}
            r = run_cpu_reference(paths, args.steps, max(args.warmup, 1), world, policy, cast)
            line = {"metric": METRIC, "value": round(r["value"], 4), "unit": "GB/s", "n_gpus": args.gpus,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["seconds"] * 1e3, 1),
                    "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype_tag,
                    "data": "synthetic", "impl": "reference",
                    "config": {"workload": workload, "global_batch": 1, "seq_len": 0, "parallelism": f"cpu, {world} thread-rank(s)"},
                    "cpu_baseline": r,
                    "e2e": {"value": round(r["value"], 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0}}
            print(json.dumps(line), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return

    from paper_2505_23072_b200 import DistGroup, LoaderConfig, SafeTensorsFileLoader, SingleGroup, _native, kernels
    from paper_2505_23072_b200.loader import FilesBufferOnDevice, _HostedFile
    from paper_2505_23072_b200.device import DeviceBuffer

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    group = DistGroup(device=device, data_plane=args.data_plane) if world > 1 else SingleGroup()
    mapping = {r: [str(p) for i, p in enumerate(paths) if i % world == r] for r in range(world)}
    keys = [e[0] for e in ents]
    policy = {e[0]: (synth.shard_dim(e[0], e[2]) if world > 1 else None) for e in ents}
    cfg = LoaderConfig(backend=args.backend, auto_release=True)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if SHARE_GPU else device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def ready_bytes_for_rank(r: int, out: bool = False) -> int:
        """Tensor body bytes rank r makes ready (its slices of sharded keys);
        out=True counts them in the retrieval dtype instead."""
        nb = 0
        for name, dt, shape in ents:
            d = policy[name]
            osz = (cast or dt).size_bytes if out else dt.size_bytes
            if d is None:
                nb += math.prod(shape) * osz
            else:
                lo, hi = kernels.shard_bounds(shape[d], world, r)
                nb += math.prod(shape) // shape[d] * (hi - lo) * osz
        return nb

    job_bytes = sum(ready_bytes_for_rank(r) for r in range(world))  # the metric: Σ tensor body bytes
    out_bytes = sum(ready_bytes_for_rank(r, out=True) for r in range(world))

    dims = {k: d for k, d in policy.items() if d is not None}

    def retrieve(fb, batched: bool):
        if batched:
            return list(fb.get_tensors(keys, dtype=cast, dims=dims).values())
        outs = []
        for k in keys:
            d = policy[k]
            outs.append(fb.get_tensor(k, dtype=cast) if d is None else fb.get_sharded(k, d, dtype=cast))
        return outs

    # ---- value leg: landed bytes in HBM -> ready tensors --------------------------------
    base_loader = SafeTensorsFileLoader(group, args.backend, rank=rank,
                                        config=LoaderConfig(backend=args.backend, auto_release=False))
    base_loader.add_filenames(mapping)
    landed = base_loader.copy_files_to_device()
    torch.cuda.synchronize()

    def fresh_fb():
        hosted = {}
        for p, hf in landed._hosted.items():
            buf = DeviceBuffer(base_loader.pool, hf.buffer.tensor, hf.buffer.capacity)
            buf.refcount = hf.unconsumed
            hosted[p] = _HostedFile(buf, dict(hf.dev_offsets), hf.unconsumed)
        base_loader.config.auto_release = True
        fb = FilesBufferOnDevice(base_loader, hosted)
        fb._peer, fb._peer_offsets = landed._peer, landed._peer_offsets  # the mapping belongs to `landed`
        return fb

    kernels.TIMING = []
    vals, dom_ms, dom_bytes = [], [], 0
    launches_value = 0
    for i in range(args.warmup + args.steps):
        fb = fresh_fb()
        barrier()
        torch.cuda.synchronize()
        kernels.TIMING.clear()
        l0 = _native.kernel_launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        outs = retrieve(fb, batched=True)
        e1.record()
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1))
        if i >= args.warmup:
            vals.append(ms)
            launches_value += _native.kernel_launches() - l0
            k_ms = sum(a.elapsed_time(b) for a, b, _ in kernels.TIMING)
            k_bytes = sum(nb for _, _, nb in kernels.TIMING)
            k_n = len(kernels.TIMING)
            # the dominant launch of the step (get_tensors issues a small head group first)
            a_, b_, nb_ = max(kernels.TIMING, key=lambda t: t[2])
            dom_ms.append(a_.elapsed_time(b_))
            dom_bytes = nb_
        del outs
        torch.cuda.synchronize()
        barrier()  # every rank is done reading peers' landed buffers
        fb._hosted, fb._peer = {}, None  # landed buffers (and their mappings) are shared across steps
        fb.close()
    kernels.TIMING = None
    value_ms = statistics.median(vals)
    value = job_bytes / (value_ms / 1e3) / 1e9
    hbm_peak, peak_source = hbm_peak_gbs()
    achieved = dom_bytes / (statistics.mean(dom_ms) / 1e3) / 1e9 if dom_ms else None
    achieved_all = k_bytes / (k_ms / 1e3) / 1e9 if k_n else None
    traffic = None
    tr_file = ROOT / "profiles" / "ncu_traffic.json"
    if tr_file.exists():
        try:
            traffic = json.loads(tr_file.read_text()).get(f"{args.arch}-{args.header}-w{world}"
                                                                + (f"-L{args.layers}" if args.layers is not None else "")
                                                                + (f"-{cast.value}" if cast else ""))
        except (OSError, ValueError):
            traffic = None
    landed.close()
    del landed
    base_loader.close()
    torch.cuda.empty_cache()

    # ---- e2e leg: files on disk -> ready tensors through the drop-in API ------------------
    def e2e_step():
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        loader = SafeTensorsFileLoader(group, args.backend, rank=rank, config=cfg)
        loader.add_filenames(mapping)
        t1 = time.perf_counter()
        fb = loader.copy_files_to_device()
        t2 = time.perf_counter()
        outs = retrieve(fb, batched=False)
        t3 = time.perf_counter()
        checksum = outs[-1].torch.reshape(-1)[:32].view(torch.uint8).cpu()  # D2H read of the result
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ms = max(e0.elapsed_time(e1), wall * 1e3)
        stats = loader.last_transfer_stats
        d2h = checksum.numel()
        phases.append({"add_filenames_ms": (t1 - t0) * 1e3, "copy_files_to_device_ms": (t2 - t1) * 1e3,
                       "engine_ms": stats.engine_seconds * 1e3 if stats else 0.0,
                       "worker_read_s": stats.read_seconds if stats else 0.0,
                       "worker_wait_s": stats.wait_seconds if stats else 0.0,
                       "retrieve_enqueue_ms": (t3 - t2) * 1e3, "drain_ms": wall * 1e3 - (t3 - t0) * 1e3})
        del outs
        fb.close()
        loader.close()
        return max_over_ranks(ms), stats, d2h

    phases = []
    clocks = Clocks(local)
    e2e_ms, launches_e2e, io_modes, h2d_bytes, ring = [], 0, set(), 0, 0.0
    first_ms = None
    warm_cache(mapping[rank])  # "warm" means resident: O_DIRECT reads of a cold file would not make it so
    host_mem = host_memory()
    resid = {"after_warm": residency(mapping[rank])}
    for i in range(args.warmup):
        ms, _, _ = e2e_step()
        if first_ms is None:
            first_ms = ms  # includes the engine's one-time pinned-ring setup and CUDA lazy init
    clocks.start()
    for i in range(args.steps):
        l0 = _native.kernel_launches()
        ms, st, d2h = e2e_step()
        e2e_ms.append(ms)
        launches_e2e += _native.kernel_launches() - l0
        if st is not None:
            io_modes.update(st.io_modes)
            h2d_bytes = st.bytes
            ring = max(ring, st.ring_setup_seconds)
    clk = clocks.stop()
    resid["after_warm_steps"] = residency(mapping[rank])
    phase_med = {k: round(statistics.median(p[k] for p in phases[-args.steps:]), 2) for k in phases[-1]}
    e2e_med = statistics.median(e2e_ms)
    e2e_val = job_bytes / (e2e_med / 1e3) / 1e9

    cold = None
    if args.cold:
        cms = []
        for i in range(max(1, min(args.steps, 2))):
            drop_cache(paths)
            ms, st, _ = e2e_step()
            cms.append(ms)
        cold = {"value": round(job_bytes / (statistics.median(cms) / 1e3) / 1e9, 3), "unit": "GB/s",
                "seconds_to_ready": round(statistics.median(cms) / 1e3, 3),
                "io_modes": sorted(st.io_modes) if st else None}

    io = None
    cpu = None
    libs = None
    views = None
    fresh = None
    if rank == 0 and world == 1 and not args.quick:
        if args.baselines and cast is None:
            # apples to apples with upstream (whose get_tensor returns views): our zero-copy mode
            cfg.auto_release = False
            warm_cache(paths)  # the cold leg left the files out of the page cache
            e2e_step()
            vms = [e2e_step()[0] for _ in range(args.steps)]
            cfg.auto_release = True
            views = {"value": round(job_bytes / (statistics.median(vms) / 1e3) / 1e9, 3), "unit": "GB/s",
                     "seconds_to_ready": round(statistics.median(vms) / 1e3, 4), "auto_release": False}
            libs = library_baselines(paths, local, tensor_bytes)
        warm_cache(paths)
        fresh = e2e_fresh_process(paths, local, args.backend, job_bytes) if cast is None else None
        if args.cpu_baseline:
            if not args.baselines:
                warm_cache(paths)
            cpu = run_cpu_reference(paths, steps=1, warmup=0, cast=cast)  # warm page cache, like the e2e leg
        io = io_probes(paths, local)  # last: it drops the first file from the page cache

    if rank == 0:
        roofline = {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None, "peak": hbm_peak,
                    "unit": "GB/s", "frac": round(achieved / hbm_peak, 4) if achieved else None,
                    "traffic": traffic,
                    "kernel": (f"hl_gather staged_kernel<{src_dt.value}->{cast.value}> (TMA in + out)" if cast
                               else "hl_gather bulk_kernel (TMA cp.async.bulk copy)"),
                    "launches_per_step": k_n, "algorithmic_bytes_per_launch": dom_bytes,
                    "achieved_all_launches_of_step": round(achieved_all, 1) if achieved_all else None,
                    # live: the kernel's share of the value step (the rest is host pre-launch work);
                    # ncu's launch list has this launch as the step's only GPU work (profiles/)
                    "kernel_share_of_step": round(k_ms / max(value_ms, 1e-9), 4) if k_n else None,
                    "peak_source": peak_source}
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(value_ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": dtype_tag, "data": "synthetic",
            "config": {"workload": workload, "cast": cast.value if cast else None,
                       "layers": args.layers, "tensor_bytes": tensor_bytes, "file_bytes": file_bytes, "ready_bytes_job": job_bytes, "ready_bytes_out": out_bytes,
                       "tensors": len(ents), "header": args.header, "backend": args.backend,
                       "auto_release": True, "global_batch": 1, "seq_len": 0,
                       "parallelism": f"tp{world}" if world > 1 else "single",
                       "data_plane": group.data_plane if world > 1 else None,
                       "l2": f"inputs ({tensor_bytes / 1e9:.1f} GB) far exceed the 126 MB L2; no flush needed"},
            "e2e": {"value": round(e2e_val, 3), "unit": "GB/s", "seconds_to_ready": round(e2e_med / 1e3, 4),
                    "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h, "page_cache": "warm",
                    "io_modes": sorted(io_modes), "ring_setup_seconds_first_load": round(ring, 4),
                    "page_cache_residency": resid, "host_memory_gb": host_mem,
                    "first_load_seconds_in_process": round(first_ms / 1e3, 4) if first_ms else None,
                    "phases_ms": phase_med},
            "e2e_cold": cold,
            "e2e_views": views,
            "e2e_fresh_process": fresh,
            "library_baselines": libs,
            "roofline": roofline,
            "io_roofline": io,
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches_e2e,
            "gpu_launches_value_leg": launches_value,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
