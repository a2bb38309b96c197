"""Device memory on a B200: backends, buffers and the accounting pool.

Reference counterpart: pkg/src/aggload/device.py (numpy byte arrays standing in
for device memory). Here a :class:`DeviceBuffer` is a ``torch.uint8`` CUDA
allocation from the torch caching allocator (the paper's "return GPU memory to
the PyTorch memory pool"); :class:`DevicePool` keeps the
reference's observable counters (allocated / pooled / cumulative pooled bytes,
a capacity cap for out-of-memory tests) on top of it. Released buffers go back
to torch's cache, which is the real pool; the counters are bookkeeping.

Backends decide where a file's bytes land in its buffer:

* ``host`` (ref DeviceBackend.host): the pinned-ring engine lands the body at
  buffer offset 0, so a tensor sits at ``data_offsets.begin`` and is aligned
  whenever the writer aligned it — no realign pass for odd-sized headers.
* ``simdirect`` (ref DeviceBackend.sim_direct): GDS-shaped landing — the
  transfer starts at the 512-byte floor of the body offset, exactly as the
  reference's direct backend, so odd headers leave tensors misaligned and the
  realign kernel repacks them (ref device.py:466-548).
* ``gds``: cuFile (GPUDirect Storage) reads straight into HBM, 4 KiB landing.

The bulk copy itself is the native engine (``_native.IoEngine``); the byte
moves after landing (realign, clone, shard pack, cast) are ``hl_gather``.
"""

from __future__ import annotations

import math
import os
import threading
import weakref
from dataclasses import dataclass
from enum import Enum

import torch

from . import _native
from .errors import (
    BounceTooSmall,
    DoubleRelease,
    IoError,
    MisalignedDirectTransfer,
    NativeUnavailable,
    OutOfBoundsView,
    OutOfMemory,
    UnsupportedConversion,
)
from .format import DType, TensorMetadata

__all__ = [
    "BackendKind",
    "DeviceBackend",
    "DeviceBuffer",
    "DevicePool",
    "DIRECT_ALIGNMENT",
    "DEFAULT_HOST_BOUNCE",
    "DEFAULT_ALIGN_BOUNCE",
    "cuda_device",
    "conversion_supported",
    "transfer_from_file",
    "align_and_convert",
    "align_fix",
    "convert_dtype",
]

DIRECT_ALIGNMENT = 512               # ref device.py:51 (simdirect landing granularity)
GDS_ALIGNMENT = 4096                 # cuFile / O_DIRECT block granularity
DEFAULT_HOST_BOUNCE = 4 * 1024 * 1024  # pinned chunk per pread + H2D hop (ref: 160 MiB host bounce; 4 MiB measured best, profiles/)
DEFAULT_ALIGN_BOUNCE = 16 * 1024 * 1024  # kept for API parity; the realign kernel needs no bounce
CARVE_CHUNK = 1 << 30                # largest shared chunk per-key outputs are carved from
CARVE_SMALL = 1 << 20                # outputs below this (norms, biases) share their own chunks...
CARVE_SMALL_CHUNK = 16 << 20         # ...of this size, so keeping one of them pins 16 MiB, not 1 GiB
CARVE_OPEN = 16                      # chunks with room left that a new output may be carved from


class BackendKind(Enum):
    HOST = "host"
    SIM_DIRECT = "simdirect"
    GDS = "gds"


@dataclass(frozen=True)
class DeviceBackend:
    """Landing rule + default I/O mode (ref device.py:61-81)."""

    kind: BackendKind
    transfer_alignment: int
    bounce_buffer_bytes: int
    io_mode: str = "auto"

    @classmethod
    def host(cls, bounce_buffer_bytes: int = DEFAULT_HOST_BOUNCE) -> "DeviceBackend":
        return cls(BackendKind.HOST, 1, bounce_buffer_bytes, "auto")

    @classmethod
    def sim_direct(cls, bounce_buffer_bytes: int = DEFAULT_ALIGN_BOUNCE) -> "DeviceBackend":
        return cls(BackendKind.SIM_DIRECT, DIRECT_ALIGNMENT, bounce_buffer_bytes, "auto")

    @classmethod
    def gds(cls, bounce_buffer_bytes: int = DEFAULT_HOST_BOUNCE) -> "DeviceBackend":
        return cls(BackendKind.GDS, GDS_ALIGNMENT, bounce_buffer_bytes, "cufile")

    @classmethod
    def of(cls, kind: "str | BackendKind | DeviceBackend") -> "DeviceBackend":
        if isinstance(kind, DeviceBackend):
            return kind
        if isinstance(kind, str):
            kind = BackendKind(kind.lower())
        if kind is BackendKind.HOST:
            return cls.host()
        if kind is BackendKind.GDS:
            return cls.gds()
        return cls.sim_direct()


def cuda_device(index: int | None = None) -> torch.device:
    """The CUDA device for a rank; refuses to run without one (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible: the load path runs only on the GPU")
    n = torch.cuda.device_count()
    idx = torch.cuda.current_device() if index is None else index % n
    return torch.device("cuda", idx)


def conversion_supported(src: DType, dst: DType) -> bool:
    return _native.conversion_supported(src.code, dst.code)


def check_conversion(src: DType, dst: DType, name: str = "") -> None:
    if not conversion_supported(src, dst):
        what = f"tensor {name!r}: " if name else ""
        raise UnsupportedConversion(f"{what}{src.value} -> {dst.value} is not supported")


class DeviceBuffer:
    """One contiguous HBM allocation: the unit of bulk transfer and release
    (ref device.py:84-130). ``tensor`` is the uint8 CUDA tensor; views made by
    tensorview.make_view alias it without copying."""

    def __init__(self, pool: "DevicePool", tensor: torch.Tensor, capacity: int):
        self.pool = pool
        self._tensor = tensor
        self.capacity = int(capacity)
        self.device_id = pool.device_id
        self.backend = pool.backend
        self.refcount = 0
        self.released = False
        self._views: weakref.WeakSet | None = None  # created with the first view (most buffers get one)
        self._pending = None  # a deferred retrieval batch that still has to write this buffer

    @property
    def tensor(self) -> torch.Tensor:
        if self.released:
            raise DoubleRelease(f"buffer on device {self.device_id} was already released")
        if self._pending is not None:
            self._pending.flush()
        return self._tensor

    # reference spelling: the raw byte array behind the buffer
    array = tensor

    @property
    def ptr(self) -> int:
        return self.tensor.data_ptr()

    def _check_range(self, off: int, length: int) -> None:
        if off < 0 or length < 0 or off + length > self.capacity:
            raise OutOfBoundsView(f"range [{off}, {off + length}) outside buffer capacity {self.capacity}")

    def write_bytes(self, off: int, data) -> None:
        raw = bytes(data) if not isinstance(data, (bytes, bytearray)) else data
        self._check_range(off, len(raw))
        if raw:
            src = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
            self.tensor[off : off + len(raw)].copy_(src)

    def read_bytes(self, off: int, length: int) -> bytes:
        self._check_range(off, length)
        if length == 0:
            return b""
        return self.tensor[off : off + length].cpu().numpy().tobytes()

    def live_view_count(self) -> int:
        return len(self._views) if self._views is not None else 0

    def _add_view(self, view) -> None:
        if self._views is None:
            self._views = weakref.WeakSet()
        self._views.add(view)

    def release(self, *, force: bool = False, to_pool: bool = True) -> None:
        self.pool.release(self, force=force, to_pool=to_pool)

    def __repr__(self) -> str:
        state = "released" if self.released else f"refcount={self.refcount}"
        return f"DeviceBuffer(cuda:{self.device_id}, capacity={self.capacity}, {state})"


class DevicePool:
    """Accounting layer over the torch caching allocator (ref device.py:133-214).

    ``allocate`` never zero-fills unless asked (every byte the loader reads was
    written by the transfer or the kernel); ``release`` drops the pool's
    reference so torch can recycle the memory, and moves the bytes from
    ``allocated_bytes`` to ``pooled_bytes``. Exact-size reuse of a pooled
    block is accounted like the reference.
    """

    def __init__(self, backend: DeviceBackend | str = "host", device_id: int | None = None,
                 capacity_cap: int | None = None):
        self.backend = DeviceBackend.of(backend)
        self.device = cuda_device(device_id)
        self.device_id = self.device.index
        self.capacity_cap = capacity_cap
        self._lock = threading.Lock()
        self._free: dict[int, int] = {}
        self.allocated_bytes = 0
        self.pooled_bytes = 0
        self.cumulative_pooled_bytes = 0
        # carving: per-key outputs sliced from shared chunks (see _carve)
        self._open: list[list] = []  # [chunk tensor, next free offset]: chunks with room left (first fit)
        self._small: torch.Tensor | None = None  # chunk for outputs under CARVE_SMALL
        self._small_off = 0
        self._expect = 0

    def expect(self, nbytes: int) -> None:
        """Announce roughly how many bytes of per-key outputs are coming
        (sizes the carving chunks)."""
        with self._lock:
            self._expect = max(0, int(nbytes))

    def end_carving(self) -> None:
        """Drop the pool's reference to the current chunk (slices keep theirs)."""
        with self._lock:
            self._open, self._expect = [], 0
            self._small, self._small_off = None, 0

    def _carve(self, nbytes: int) -> torch.Tensor:
        """A 256-byte aligned slice of a shared chunk. A fresh process pays
        one cudaMalloc per torch caching-allocator segment; carving the ~300
        per-key outputs of a checkpoint out of a few chunks (each sized by the
        announced remaining bytes, at most CARVE_CHUNK) turns a first load's
        ~1 s of allocator growth into a few calls. Accounting stays per buffer;
        a chunk's memory returns when its last slice dies — so a caller that
        keeps one output alive keeps its whole chunk resident: at most
        CARVE_CHUNK (and never more than the handle's announced outputs) for a
        weight, CARVE_SMALL_CHUNK for an output under CARVE_SMALL (norms and
        biases are carved apart from the weights). With a ``capacity_cap``
        nothing is carved (``allocate``)."""
        if nbytes < CARVE_SMALL:
            # small outputs get their own chunks: a caller that keeps only a few norms
            # or biases then pins CARVE_SMALL_CHUNK, not a big chunk of weights
            if self._small is None or self._small_off + nbytes > self._small.numel():
                self._small = torch.empty(CARVE_SMALL_CHUNK, dtype=torch.uint8, device=self.device)
                self._small_off = 0
            t = self._small[self._small_off:self._small_off + nbytes]
            self._small_off += (nbytes + 255) & ~255
            return t
        # first fit over the chunks that still have room: big weights (a 70B MLP matrix is
        # 470 MB of a 1 GiB chunk) leave gaps that later, smaller outputs fill; carving only
        # from the newest chunk wasted 25-33% of HBM on 70B (profiles/r02_carve_fit.txt)
        for ent in self._open:
            if ent[1] + nbytes <= ent[0].numel():
                break
        else:
            size = max(nbytes, min(CARVE_CHUNK, max(self._expect, nbytes)))
            ent = [torch.empty(size, dtype=torch.uint8, device=self.device), 0]
            self._open.append(ent)
        t = ent[0][ent[1]:ent[1] + nbytes]
        ent[1] += (nbytes + 255) & ~255
        self._expect = max(0, self._expect - nbytes)
        # chunks with less than a small output's room left are closed (the list stays short)
        self._open = [e for e in self._open if e[0].numel() - e[1] >= CARVE_SMALL][-CARVE_OPEN:]
        return t

    def allocate(self, size: int, zero: bool = False, carve: bool = False) -> DeviceBuffer:
        if size < 0:
            raise ValueError(f"allocation size must be non-negative, got {size}")
        with self._lock:
            if self._free.get(size):
                self._free[size] -= 1
                self.pooled_bytes -= size
            else:
                if self.capacity_cap is not None:
                    while self.allocated_bytes + self.pooled_bytes + size > self.capacity_cap and self.pooled_bytes > 0:
                        self._evict_one()
                    if self.allocated_bytes + size > self.capacity_cap:
                        raise OutOfMemory(
                            f"device {self.device_id}: {size} bytes requested, "
                            f"{self.allocated_bytes} live of {self.capacity_cap} cap")
            try:
                # +16: 16-byte vector loads of a tensor's last bytes stay inside the allocation.
                # Carving is off under a capacity cap: a chunk is device memory the cap's
                # accounting (requested sizes) would not see.
                if carve and self.capacity_cap is None:
                    try:
                        t = self._carve(max(size, 1) + 16)
                    except torch.OutOfMemoryError:
                        self._open = []
                        self._small, self._small_off = None, 0
                        t = torch.empty(max(size, 1) + 16, dtype=torch.uint8, device=self.device)
                else:
                    t = torch.empty(max(size, 1) + 16, dtype=torch.uint8, device=self.device)
            except torch.OutOfMemoryError as e:
                raise OutOfMemory(f"device {self.device_id}: cannot allocate {size} bytes: {e}") from None
            if zero:
                t.zero_()
            self.allocated_bytes += size
            return DeviceBuffer(self, t, size)

    def _evict_one(self) -> None:
        for cap in sorted(self._free):
            if self._free[cap]:
                self._free[cap] -= 1
                self.pooled_bytes -= cap
                return

    def release(self, buf: DeviceBuffer, *, force: bool = False, to_pool: bool = True) -> None:
        with self._lock:
            if buf.released:
                raise DoubleRelease(f"buffer on device {self.device_id} released twice")
            if not force:
                if buf.refcount != 0:
                    raise ValueError(f"buffer still hosts {buf.refcount} unconsumed keys; only close may force it")
                if buf.live_view_count() > 0:
                    raise ValueError(f"buffer has {buf.live_view_count()} live views; only close may force it")
            buf.released = True
            self.allocated_bytes -= buf.capacity
            if to_pool:
                self._free[buf.capacity] = self._free.get(buf.capacity, 0) + 1
                self.pooled_bytes += buf.capacity
                self.cumulative_pooled_bytes += buf.capacity
            buf._tensor = None  # torch's caching allocator takes it back once views die


# ---------------------------------------------------------------- device sub-boundary
# The reference's device backend also exposes its building blocks one call at a
# time (ref device.py:238-590): a ranged file -> device transfer, the realign
# repack, and an in-place dtype conversion. The loader never calls these (it
# lands whole files through the engine and realigns out of place in one batched
# launch, loader.py _land); they exist so code written against the reference's
# device module keeps working, with the same arguments, results and errors, on
# the same engine and kernel as the hot path.

def _path_of(file) -> str:
    """A readable path for the engine: an fd or file object (the reference's
    ``_fd_of`` inputs, ref device.py:220-223) resolves through /proc."""
    if isinstance(file, (str, bytes)) or hasattr(file, "__fspath__"):
        return os.fsdecode(file)
    fd = file if isinstance(file, int) else file.fileno()
    return os.readlink(f"/proc/self/fd/{fd}")


def transfer_from_file(buf: DeviceBuffer, dev_off: int, file, file_off: int, length: int,
                       staging=None) -> None:
    """Copy ``length`` file bytes at ``file_off`` into ``buf`` at ``dev_off``
    (ref device.py:238-288): bounds, the direct backends' alignment rule (offsets
    and length multiples of the landing granularity unless the range ends at
    end-of-file: MisalignedDirectTransfer), IoError on a short file. The bytes
    move through the native engine's pinned ring (``hl_transfer_from_file``);
    ``staging`` is accepted for signature parity — the ring is the staging — and
    a zero-capacity one raises BounceTooSmall as in the reference."""
    from .transfer import engine_for, engine_team  # transfer imports this module

    buf._check_range(dev_off, length)
    path = _path_of(file)
    if length == 0:
        return
    kind = buf.backend.kind
    if kind is not BackendKind.HOST:
        align = buf.backend.transfer_alignment
        if file_off % align or dev_off % align:
            raise MisalignedDirectTransfer(f"direct transfer needs {align}-byte aligned offsets, "
                                           f"got file_off={file_off} dev_off={dev_off}")
        if length % align and file_off + length != os.stat(path).st_size:
            raise MisalignedDirectTransfer(f"direct transfer length {length} is not a {align} multiple "
                                           "and does not end at end-of-file")
    elif staging is not None and min(buf.backend.bounce_buffer_bytes, getattr(staging, "nbytes", len(staging))) <= 0:
        raise BounceTooSmall("host staging buffer has zero capacity")
    if file_off + length > os.stat(path).st_size:
        raise IoError(f"unexpected EOF: [{file_off}, {file_off + length}) past the end of {path}")
    eng = engine_for(buf.device_id, engine_team(), buf.backend.bounce_buffer_bytes, buf.backend.io_mode)
    with torch.cuda.device(buf.device_id):
        eng.transfer(path, file_off, length, buf.ptr + dev_off,
                     after_stream=torch.cuda.current_stream(buf.device_id).cuda_stream)


def _scratch_rewrite(buf: DeviceBuffer, end: int, descs_into) -> None:
    """Rewrite ``buf[0:end)`` in place without the reference's overlap-ordered
    chunk moves: snapshot the region, let ``descs_into(scratch_ptr)`` build the
    moves from the ORIGINAL bytes into the snapshot, copy it back. Bytes no move
    writes (alignment padding, a narrowed tail) keep their old values, exactly as
    the reference's in-place moves leave them. Three hl_gather launches on the
    current stream."""
    from . import kernels  # kernels is a leaf module; imported lazily to keep this one light

    dev = torch.device("cuda", buf.device_id)
    scratch = torch.empty(max(end, 1), dtype=torch.uint8, device=dev)
    kernels.run([kernels.copy_desc(buf.ptr, scratch.data_ptr(), end, DType.U8)], dev)
    kernels.run(descs_into(scratch.data_ptr()), dev)
    kernels.run([kernels.copy_desc(scratch.data_ptr(), buf.ptr, end, DType.U8)], dev)


def align_and_convert(buf: DeviceBuffer, landing, bounce: int, conversions: dict | None = None) -> list:
    """Repack tensors to dtype-aligned offsets, converting dtypes in the same
    pass (ref device.py:466-534): ascending landing order, each start rounded up
    to the (target) dtype's alignment; a no-op returning the landing offsets
    when nothing converts and everything is aligned. Errors as the reference:
    UnsupportedConversion, OutOfBoundsView when the repacked layout outgrows the
    buffer, BounceTooSmall when ``bounce`` cannot hold one element (the kernel
    needs no bounce; the check keeps the contract). Returns
    ``[(name, new_offset, TensorMetadata)]``."""
    from . import kernels

    conversions = conversions or {}
    entries = sorted(landing, key=lambda e: e[1])
    for name, _, meta in entries:
        target = conversions.get(name, meta.dtype)
        if target is not meta.dtype:
            check_conversion(meta.dtype, target, name)
    if not conversions and all(off % meta.dtype.alignment == 0 for _, off, meta in entries):
        return [(name, off, TensorMetadata(meta.name, meta.dtype, meta.shape, (off, off + meta.nbytes)))
                for name, off, meta in entries]
    moves, cursor = [], 0
    for name, off, meta in entries:
        buf._check_range(off, meta.nbytes)
        dst = conversions.get(name, meta.dtype)
        numel = math.prod(meta.shape)
        dst_off = -(-cursor // dst.alignment) * dst.alignment
        moves.append((name, off, dst_off, numel, meta, dst))
        cursor = dst_off + numel * dst.size_bytes
    if cursor > buf.capacity:
        raise OutOfBoundsView(f"repacked layout needs {cursor} bytes but buffer capacity is {buf.capacity}")
    max_elem = max((max(m[4].dtype.size_bytes, m[5].size_bytes) for m in moves), default=1)
    if bounce < max_elem:
        raise BounceTooSmall(f"bounce of {bounce} bytes cannot hold a {max_elem}-byte element")
    src = buf.ptr
    _scratch_rewrite(buf, cursor, lambda out: [
        kernels.copy_desc(src + off, out + dst_off, numel, meta.dtype, dst)
        for _, off, dst_off, numel, meta, dst in moves])
    return [(name, dst_off, TensorMetadata(meta.name, dst, meta.shape, (dst_off, dst_off + numel * dst.size_bytes)))
            for name, _, dst_off, numel, meta, dst in moves]


def align_fix(buf: DeviceBuffer, landing, bounce: int = DEFAULT_ALIGN_BOUNCE) -> list:
    """Repack so every offset is dtype-aligned; idempotent (ref device.py:537-548)."""
    return [(name, off) for name, off, _ in align_and_convert(buf, landing, bounce)]


def convert_dtype(buf: DeviceBuffer, view_meta: TensorMetadata, target: DType,
                  bounce: int = DEFAULT_ALIGN_BOUNCE) -> TensorMetadata:
    """Convert one tensor region in place, keeping its begin offset
    (ref device.py:551-590); same checks and error classes as the reference."""
    from . import kernels

    check_conversion(view_meta.dtype, target)
    numel = math.prod(view_meta.shape)
    begin = view_meta.begin
    dst_bytes = numel * target.size_bytes
    if begin % target.alignment:
        raise OutOfBoundsView(f"offset {begin} is not aligned for {target.value}")
    if begin + dst_bytes > buf.capacity:
        raise OutOfBoundsView(f"converted tensor needs [{begin}, {begin + dst_bytes}) but capacity is {buf.capacity}")
    if bounce < max(view_meta.dtype.size_bytes, target.size_bytes):
        raise BounceTooSmall(f"bounce of {bounce} bytes cannot hold one element")
    if begin < 0 or begin + view_meta.nbytes > buf.capacity:
        raise OutOfBoundsView(f"tensor [{begin}, {begin + view_meta.nbytes}) outside capacity {buf.capacity}")
    src = buf.ptr + begin
    end = max(begin + dst_bytes, begin + view_meta.nbytes)
    _scratch_rewrite(buf, end, lambda out: [kernels.copy_desc(src, out + begin, numel, view_meta.dtype, target)])
    return TensorMetadata(view_meta.name, target, view_meta.shape, (begin, begin + dst_bytes))
