"""Descriptor builders over ``hl_gather`` (the batched realign/shard/cast kernel).

Every byte move after landing goes through here, enqueued on the caller's
current CUDA stream with no host synchronisation:

* :func:`copy_desc`  — whole tensor, optionally cast (clone / realign / convert),
* :func:`shard_desc` — rank slice ``[lo, hi)`` along ``dim`` of a row-major
  tensor, optionally cast (ref collective.py:318-330 ``_clone_slice``; the
  reference's oracle is reference.py:56-66 ``load_shard_bytes``),
* :func:`run`        — launch a batch (one launch per conversion kind present).
"""

from __future__ import annotations

import math
import os

import torch

from . import _native
from .format import DType

Desc = tuple  # (src, dst, rows, row_elems, src_pitch, src_code, dst_code)


def copy_desc(src_ptr: int, dst_ptr: int, numel: int, src: DType, dst: DType | None = None) -> Desc:
    dst = dst or src
    return (src_ptr, dst_ptr, 1 if numel else 0, numel, numel * src.size_bytes, src.code, dst.code)


def shard_bounds(extent: int, world: int, rank: int) -> tuple[int, int]:
    """Remainder-to-lower-ranks split (ref collective.py:62-67)."""
    base, extra = divmod(extent, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_desc(src_ptr: int, shape: tuple[int, ...], dim: int, lo: int, hi: int, dst_ptr: int,
               src: DType, dst: DType | None = None) -> Desc:
    dst = dst or src
    outer = math.prod(shape[:dim])
    inner = math.prod(shape[dim + 1:])
    ss = src.size_bytes
    rows = outer if (hi > lo and inner) else 0
    return (src_ptr + lo * inner * ss, dst_ptr, rows, (hi - lo) * inner, shape[dim] * inner * ss,
            src.code, dst.code)


def current_stream_ptr(device: torch.device) -> int:
    return _raw_stream(device.index)


# Peer pulls (sources in another GPU's memory) run on the LDG/STG warp kernels
# unless HL_PEER_TMA=1 sends them through the TMA kernels too (the TMA unit then
# issues the NVLink reads; untested on NVLink here: every gpurun box has one GPU).
PEER_TMA = os.environ.get("HL_PEER_TMA") == "1"

# Optional launch timing (bench.py): when a list, every run() appends its
# algorithmic bytes, and hl_gather records a CUDA event pair on the launch
# stream around that call's kernel launches (after the host-side descriptor
# translation); timings() pairs them up once the work is done.
TIMING: list | None = None


def timings() -> list[tuple[float, int]]:
    """(milliseconds, algorithmic bytes) of every run() since TIMING was
    (re)started, in order; clears both. Waits for the launches to finish."""
    ms = _native.gather_timings()
    nb = list(TIMING or [])
    if TIMING is not None:
        TIMING.clear()
    if len(ms) != len(nb):
        raise RuntimeError(f"launch timing: {len(ms)} event pairs for {len(nb)} runs")
    return list(zip(ms, nb))

_SIZE = [1, 1, 1, 2, 2, 4, 4, 8, 8, 2, 2, 4, 8]


def algorithmic_bytes(descs: list[Desc]) -> int:
    """Bytes a batch must move: source elements read + destination written."""
    return sum(d[2] * d[3] * (_SIZE[d[5]] + _SIZE[d[6]]) for d in descs)


try:  # the raw cudaStream_t of the device's current stream, without building a Stream object
    _raw_stream = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover
    def _raw_stream(index: int) -> int:
        return torch.cuda.current_stream(index).cuda_stream


def run(descs: list[Desc], device: torch.device, peer: bool = False, stream_ptr: int | None = None) -> None:
    """Enqueue the batch on ``device``'s current stream (or on ``stream_ptr``,
    a cudaStream_t of that device). hl_gather launches on the CURRENT device
    (grid sizing and the launch itself), so switch to the stream's device when
    the caller's differs. ``peer``: some sources are another GPU's memory (peer
    pulls) — keep them on the LDG/STG kernels."""
    if not descs:
        return
    if torch.cuda.current_device() != device.index:
        with torch.cuda.device(device):
            return run(descs, device, peer, stream_ptr)
    flags = _native.GATHER_NO_TMA if (peer and not PEER_TMA) else 0
    if TIMING is None:
        _native.gather(descs, _raw_stream(device.index) if stream_ptr is None else stream_ptr, flags)
        return
    _native.gather(descs, _raw_stream(device.index) if stream_ptr is None else stream_ptr, flags)
    TIMING.append(algorithmic_bytes(descs))
