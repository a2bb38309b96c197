"""Rank groups and the broadcast / scatter shuffle (ref pkg/src/aggload/collective.py).

Two interchangeable group types serve the loader:

* :class:`DistGroup` — the production path: one process per GPU over
  ``torch.distributed`` (NCCL on NVLink 5 / NVSwitch). ``get_tensor`` is an
  ``ncclBroadcast`` from the owner; ``get_sharded`` is one owner-side pack
  kernel (all W shards, cast fused, in a single ``hl_gather`` launch) followed
  by one grouped send/recv (``batch_isend_irecv``: ncclGroupStart/End, so
  uneven remainder parts need no padding). Everything is
  enqueued on the current stream: no host rendezvous per key. NCCL's ordering
  contract replaces the reference's descriptor-checked rendezvous; with
  ``check_order=True`` every collective first all-gathers its (op, key, src,
  dim) descriptor and a disagreement raises ``RendezvousTimeout`` like the
  reference (collective.py:149-159).
* :class:`ProcessGroup` — the reference's in-process group contract (ranks
  are threads; here they meet at per-rank mailboxes behind a two-phase
  ``threading.Barrier`` that stays broken — poisoned — after a timeout,
  abort or ordering mismatch), kept so reference-style multi-rank tests run
  unchanged on one GPU. Its data moves are ``hl_gather`` kernels reading the owner's buffer.

Partitioning (``partition``/``ShardSpec``) is the reference's arithmetic:
equal parts, the first ``shape[dim] % W`` ranks get one more (ref 52-74).
"""

from __future__ import annotations

import hashlib
import math
import threading
from dataclasses import dataclass

import torch

from . import kernels
from .errors import BadDim, DimTooSmall, RendezvousTimeout, SpecMismatch
from .format import DType, TensorMetadata

__all__ = ["ProcessGroup", "SingleGroup", "DistGroup", "ShardSpec", "partition"]

DEFAULT_TIMEOUT = 30.0
_BARRIER_SEQ: dict[tuple[str, str], int] = {}  # DistGroup.bounded_barrier calls so far, per member set
_BARRIER_LOCK = threading.Lock()


@dataclass(frozen=True)
class ShardSpec:
    key: str
    dim: int
    world_size: int
    full_shape: tuple[int, ...]
    part_shapes: tuple[tuple[int, ...], ...]

    def bounds(self, rank: int) -> tuple[int, int]:
        lo = sum(p[self.dim] for p in self.part_shapes[:rank])
        return lo, lo + self.part_shapes[rank][self.dim]

    def to_json(self) -> dict:
        return {"key": self.key, "dim": self.dim, "world_size": self.world_size,
                "full_shape": list(self.full_shape), "part_shapes": [list(p) for p in self.part_shapes]}


def partition(meta: TensorMetadata, dim: int, world_size: int) -> ShardSpec:
    shape = tuple(meta.shape)
    if dim < 0 or dim >= len(shape):
        raise BadDim(f"dim {dim} out of range for shape {list(shape)}")
    if shape[dim] < world_size:
        raise DimTooSmall(f"cannot split dim {dim} of size {shape[dim]} across {world_size} ranks")
    parts = []
    for r in range(world_size):
        lo, hi = kernels.shard_bounds(shape[dim], world_size, r)
        p = list(shape)
        p[dim] = hi - lo
        parts.append(tuple(p))
    return ShardSpec(meta.name, dim, world_size, shape, tuple(parts))


# ------------------------------------------------------------------------ data moves
def _fresh(pool, name: str, dtype: DType, shape: tuple[int, ...]):
    from .tensorview import make_view

    n = 1
    for d in shape:
        n *= d
    nb = n * dtype.size_bytes
    buf = pool.allocate(nb, carve=True)  # per-key outputs: carved from shared chunks
    return buf, make_view(buf, 0, TensorMetadata(name, dtype, tuple(shape), (0, nb)))


def clone_full(view, pool, name: str, dtype: DType | None = None):
    """A fresh tensor in ``pool`` with ``view``'s bytes, optionally cast
    (ref collective.py:313-315 and loader.py:490-499)."""
    dtype = dtype or view.dtype
    buf, out = _fresh(pool, name, dtype, view.shape)
    src_ptr, peer = _source_ptr(view, pool.device)
    kernels.run([kernels.copy_desc(src_ptr, buf.ptr, view.numel, view.dtype, dtype)], pool.device, peer)
    return buf, out


def clone_slice(view, dim: int, lo: int, hi: int, part_shape, pool, name: str, dtype: DType | None = None):
    """A fresh contiguous copy of ``view[..., lo:hi, ...]`` along ``dim``
    (ref collective.py:318-330), optionally cast in the same pass."""
    dtype = dtype or view.dtype
    buf, out = _fresh(pool, name, dtype, part_shape)
    src_ptr, peer = _source_ptr(view, pool.device)
    kernels.run([kernels.shard_desc(src_ptr, view.shape, dim, lo, hi, buf.ptr, view.dtype, dtype)], pool.device, peer)
    return buf, out


def _source_ptr(view, device: torch.device) -> tuple[int, bool]:
    """Device address of ``view`` readable from ``device``, and whether it is
    another GPU's memory. Another GPU of the same process is read in place
    over NVLink (peer access), so the kernel on the receiving GPU does the
    transfer and the slice/cast in one pass."""
    src_dev = view.buffer.tensor.device
    if src_dev != device:
        from . import _native

        _native.enable_peer_access(device.index, src_dev.index)
    return view.buffer.ptr + view.base_offset, src_dev != device


def pack_parts(spec: ShardSpec, src_ptr: int, in_dtype: DType, out_dtype: DType, own: int,
               own_out: torch.Tensor, device: torch.device, src_bytes: torch.Tensor | None = None) -> list[torch.Tensor]:
    """Owner-side pack of the NCCL scatter: every rank's slice of the tensor at
    ``src_ptr`` (cast to ``out_dtype``) with ONE hl_gather launch — the owner's
    own slice straight into ``own_out``, the others into one pack buffer with
    16-byte aligned parts. A part that is one contiguous range of the source
    (dim 0, or only size-1 dims before ``dim``) with no cast is sent straight
    from the source bytes (``src_bytes``: a uint8 tensor starting at
    ``src_ptr``), as SURVEY §8e specifies: no pack copy. Returns the W uint8
    parts, enqueued on the current stream (ref collective.py:214-255 / 318-330)."""
    esz = out_dtype.size_bytes
    sizes = [math.prod(p) * esz for p in spec.part_shapes]
    contiguous = math.prod(spec.full_shape[:spec.dim]) == 1 and in_dtype is out_dtype and src_bytes is not None
    inner = math.prod(spec.full_shape[spec.dim + 1:]) * in_dtype.size_bytes
    packed = [r for r in range(spec.world_size) if r != own and not contiguous]
    pack_bytes = sum(-(-sizes[r] // 16) * 16 for r in packed)
    pack = torch.empty(pack_bytes + 16, dtype=torch.uint8, device=device) if packed else None
    parts, descs, cursor = [], [], 0
    for r in range(spec.world_size):
        lo, hi = spec.bounds(r)
        if r == own:
            dst, part = own_out.data_ptr(), own_out
        elif contiguous:
            parts.append(src_bytes[lo * inner:lo * inner + sizes[r]])
            continue
        else:
            dst, part = pack.data_ptr() + cursor, pack[cursor : cursor + sizes[r]]
            cursor += -(-sizes[r] // 16) * 16  # keep every part 16-byte aligned
        descs.append(kernels.shard_desc(src_ptr, spec.full_shape, spec.dim, lo, hi, dst, in_dtype, out_dtype))
        parts.append(part)
    kernels.run(descs, device)
    return parts


# ------------------------------------------------------------------------ thread group
@dataclass(frozen=True)
class _Span:
    """What crosses rank threads: a region descriptor, never the view object
    (so the owner's live-view accounting is not held by peers; ref 265-283)."""

    buffer: object
    base_offset: int
    dtype: DType
    shape: tuple[int, ...]

    @property
    def numel(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    @property
    def nbytes(self) -> int:
        return self.numel * self.dtype.size_bytes


def _span_of(view) -> "_Span | None":
    return None if view is None else _Span(view.buffer, view.base_offset, view.dtype, tuple(view.shape))


class _Mailboxes:
    """The meeting point of W thread-ranks: one mailbox slot per rank and a
    two-phase ``threading.Barrier``. A round is: post into your slot, pass
    phase 1 (every slot is now written), snapshot all slots, pass phase 2
    (every rank has its snapshot, so slots may be overwritten by the next
    round). A barrier that breaks — a rank waited longer than the timeout, or
    someone aborted — stays broken: the group is poisoned and the recorded
    reason is what every later call raises."""

    def __init__(self, world_size: int):
        self._barrier = threading.Barrier(world_size)
        self._slots: list[object] = [None] * world_size
        self._posted = [False] * world_size
        self._lock = threading.Lock()
        self.reason: str | None = None

    def fail(self, reason: str) -> RendezvousTimeout:
        with self._lock:
            if self.reason is None:
                self.reason = reason
        self._barrier.abort()
        return RendezvousTimeout(self.reason)

    def _pass(self, rank: int, timeout: float, phase: str) -> None:
        try:
            self._barrier.wait(timeout)
        except threading.BrokenBarrierError:
            raise self.fail(f"rank {rank} timed out after {timeout}s at the {phase} barrier: "
                            "a peer rank failed to arrive") from None

    def round(self, rank: int, payload: object, timeout: float) -> dict[int, object]:
        with self._lock:
            if self.reason is not None:
                raise RendezvousTimeout(self.reason)
            twice = self._posted[rank]
            self._posted[rank] = True
        if twice:  # this rank is already inside a collective on another thread
            raise self.fail(f"rank {rank} issued a collective out of turn")
        self._slots[rank] = payload
        try:
            self._pass(rank, timeout, "arrive")
            snapshot = dict(enumerate(self._slots))
            self._pass(rank, timeout, "leave")
        finally:
            with self._lock:
                self._posted[rank] = False
        return snapshot


class ProcessGroup:
    """In-process ranks (threads) with blocking collectives — the reference's
    group contract (ref collective.py:77-256): ``exchange`` returns every
    rank's payload on every rank, collectives carry an (op, tag, src)
    descriptor that must agree across ranks, and a timeout, an abort or a
    descriptor disagreement poisons the group for good (``RendezvousTimeout``).
    The data moves are hl_gather kernels reading the owner's buffer."""

    def __init__(self, world_size: int, timeout: float = DEFAULT_TIMEOUT):
        if world_size < 1:
            raise ValueError(f"world_size must be >= 1, got {world_size}")
        self.world_size = world_size
        self.timeout = timeout
        self._boxes = _Mailboxes(world_size)

    def rank_ids(self) -> range:
        return range(self.world_size)

    def exchange(self, rank: int, payload: object) -> dict[int, object]:
        if not 0 <= rank < self.world_size:
            raise ValueError(f"rank {rank} not in group of {self.world_size}")
        if self.world_size == 1:
            return {0: payload}
        return self._boxes.round(rank, payload, self.timeout)

    def _checked_exchange(self, rank: int, desc: tuple, data: object) -> dict[int, object]:
        """One round carrying (descriptor, data); every rank compares all
        descriptors, so a mismatch is seen — and raised — on every rank."""
        got = self.exchange(rank, (desc, data))
        others = {d for d, _ in got.values() if d != desc}
        if others:
            raise self._boxes.fail(f"collective mismatch across ranks (ordering bug): rank {rank} issued "
                                   f"{desc}, peers issued {sorted(others | {desc}, key=repr)}")
        return {r: x for r, (_, x) in got.items()}

    def abort(self, reason: str) -> None:
        self._boxes.fail(reason)

    def agree(self, rank: int, src: int, value: object, tag: str = "") -> object:
        if self.world_size == 1:
            return value
        return self._checked_exchange(rank, ("agree", tag, src), value if rank == src else None)[src]

    def _finish(self, pool) -> None:
        # receivers' kernels read the owner's buffer: complete them before the
        # owner may consume (release) it
        if pool is not None:
            torch.cuda.current_stream(pool.device).synchronize()

    def broadcast(self, rank: int, view, src: int, pool=None, tag: str = "", meta=None):
        if not 0 <= src < self.world_size:
            raise ValueError(f"src {src} not in group of {self.world_size}")
        if self.world_size == 1:
            if view is None:
                raise SpecMismatch("broadcast source holds no view")
            return view
        if rank == src and view is not None:
            torch.cuda.current_stream(view.buffer.tensor.device).synchronize()
        payload = _span_of(view) if rank == src else None
        span = self._checked_exchange(rank, ("broadcast", tag, src), payload)[src]
        if span is None:
            raise SpecMismatch(f"broadcast src rank {src} holds no view (tag={tag!r})")
        if rank == src:
            result = view
        else:
            if pool is None:
                raise ValueError("non-source ranks need a destination pool")
            _, result = clone_full(span, pool, tag or "broadcast")
        self._finish(pool)
        self._checked_exchange(rank, ("broadcast-done", tag, src), None)
        return result

    def scatter(self, rank: int, spec: ShardSpec, src: int, source_view=None, pool=None, tag: str = "",
                dtype: DType | None = None, src_dtype: DType | None = None):
        if spec.world_size != self.world_size:
            raise SpecMismatch(f"spec is for world {spec.world_size}, group is {self.world_size}")
        if self.world_size == 1:
            if source_view is None:
                raise SpecMismatch("scatter source holds no view")
            return source_view
        if rank == src and source_view is not None:
            torch.cuda.current_stream(source_view.buffer.tensor.device).synchronize()
        payload = _span_of(source_view) if rank == src else None
        span = self._checked_exchange(rank, ("scatter", tag, src, spec.dim, spec.full_shape), payload)[src]
        if span is None:
            raise SpecMismatch(f"scatter src rank {src} holds no view (tag={tag!r})")
        if span.shape != spec.full_shape:
            raise SpecMismatch(f"source shape {list(span.shape)} does not match spec {list(spec.full_shape)}")
        if pool is None:
            raise ValueError("scatter needs a destination pool on every rank")
        lo, hi = spec.bounds(rank)
        _, result = clone_slice(span, spec.dim, lo, hi, spec.part_shapes[rank], pool,
                                tag or spec.key, dtype)
        self._finish(pool)
        self._checked_exchange(rank, ("scatter-done", tag, src), None)
        return result


class SingleGroup(ProcessGroup):
    """World of one (ref collective.py:258-262)."""

    def __init__(self):
        super().__init__(1)


# ------------------------------------------------------------------------ torch.distributed
class DistGroup:
    """One process per GPU over ``torch.distributed`` (NCCL on GPUs, gloo on CPU).

    ``rank`` arguments are group ranks, as in :class:`ProcessGroup`, so the
    loader drives both group types through the same calls.
    """

    def __init__(self, group=None, device: torch.device | None = None, check_order: bool = False,
                 timeout: float = DEFAULT_TIMEOUT, data_plane: str = "auto"):
        import torch.distributed as dist

        if data_plane not in ("auto", "nccl", "ipc"):
            raise ValueError(f"unknown data plane {data_plane!r}")

        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self._dist = dist
        self.pg = group
        self.world_size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.timeout = timeout
        self.check_order = check_order
        self.backend = dist.get_backend(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if self.backend == "nccl" else torch.device("cpu")
        self.device = torch.device(device)
        if data_plane == "auto":
            # peer memory (CUDA IPC) needs every rank on one node and on GPUs
            import socket

            hosts = self.exchange(self.rank, socket.gethostname()) if self.world_size > 1 else {0: ""}
            one_node = len(set(hosts.values())) == 1
            data_plane = "ipc" if (one_node and self.device.type == "cuda") else "nccl"
            if data_plane == "ipc" and self.world_size > 1 and not self._ipc_works():
                data_plane = "nccl"  # e.g. a container without IPC rights: the same path over NCCL
        self.data_plane = data_plane

    def rank_ids(self) -> range:
        return range(self.world_size)

    def _ipc_works(self) -> bool:
        """Probe the peer-memory plane once: every rank maps its right
        neighbour's allocation through CUDA IPC and reads it with one hl_gather
        launch. Collective; True only if it worked on every rank."""
        from . import _native

        probe = torch.full((4096,), (self.rank + 1) % 256, dtype=torch.uint8, device=self.device)
        torch.cuda.synchronize(self.device)
        try:
            mine = _native.ipc_export(probe.data_ptr())
        except Exception:  # noqa: BLE001 - any failure means: use NCCL
            mine = None
        handles = self.exchange(self.rank, mine)
        peer = (self.rank + 1) % self.world_size
        ok, ptr = False, None
        try:
            if handles[peer] is not None:
                ptr = _native.ipc_import(handles[peer], self.device.index)
                out = torch.zeros(4096, dtype=torch.uint8, device=self.device)
                kernels.run([kernels.copy_desc(ptr, out.data_ptr(), 4096, DType.U8)], self.device, peer=True)
                torch.cuda.synchronize(self.device)
                ok = bool((out == (peer + 1) % 256).all().item())
        except Exception:  # noqa: BLE001
            ok = False
        finally:
            if ptr is not None:
                _native.ipc_release(ptr)
        verdict = all(self.exchange(self.rank, ok).values())  # also keeps every probe alive until read
        del probe
        return verdict

    # -- peer-memory data plane ("ipc") --------------------------------------------------
    def publish(self, buffers: dict[str, int], device_index: int) -> dict[str, int]:
        """Exchange the HBM addresses of every rank's landed file buffers.

        ``buffers`` maps this rank's file ids to device pointers (bytes already
        final on the device: the caller synchronised its stream). Returns
        ``file id -> pointer usable on this rank`` for ALL files: its own as
        given, every peer's opened through CUDA IPC. One collective per load.
        """
        from . import _native

        mine = {f: _native.ipc_export(p) for f, p in buffers.items()}
        out = dict(buffers)
        if self.world_size == 1:
            return out
        for r, theirs in self.exchange(self.rank, mine).items():
            if r == self.rank:
                continue
            for f, h in theirs.items():
                out[f] = _native.ipc_import(h, device_index)
        return out

    def unpublish(self, imported: dict[str, int], own: set[str]) -> None:
        """Close peer mappings, then wait until every rank did, so owners may
        free the memory. A collective, bounded by ``timeout``: a rank that never
        closes makes the others raise RendezvousTimeout instead of hanging."""
        from . import _native

        for f, p in imported.items():
            if f not in own:
                _native.ipc_release(p)
        self.bounded_barrier("unpublish")

    def bounded_barrier(self, tag: str, timeout: float | None = None) -> None:
        """Barrier through the rendezvous store (a counter per call) that gives
        up after ``timeout`` seconds (default: the group's) with
        RendezvousTimeout — unlike a NCCL/gloo barrier, it cannot hang an
        error path until the watchdog fires."""
        if self.world_size == 1:
            return
        import time

        from torch.distributed import distributed_c10d as c10d

        store = c10d._get_default_store()
        members = "all" if self.pg is None else ",".join(map(str, c10d.get_process_group_ranks(self.pg)))
        # the sequence number is per process and member set, not per DistGroup object: a later
        # group over the same ranks must not meet at keys an earlier one already filled
        with _BARRIER_LOCK:
            seq = _BARRIER_SEQ[(members, tag)] = _BARRIER_SEQ.get((members, tag), 0) + 1
        key = f"hl-barrier/{members}/{tag}/{seq}"
        limit = self.timeout if timeout is None else timeout
        deadline = time.monotonic() + limit
        arrived = store.add(key, 1)
        pause = 1e-4
        while arrived < self.world_size:
            if time.monotonic() > deadline:
                raise RendezvousTimeout(f"rank {self.rank}: {arrived} of {self.world_size} ranks reached "
                                        f"{tag!r} within {limit}s")
            time.sleep(pause)
            pause = min(pause * 2, 0.01)
            arrived = store.add(key, 0)

    def barrier(self) -> None:
        if self.world_size > 1:
            self._dist.barrier(group=self.pg)

    def _global(self, r: int) -> int:
        return r if self.pg is None else self._dist.get_global_rank(self.pg, r)

    # -- control plane ---------------------------------------------------------------
    def exchange(self, rank: int, payload: object) -> dict[int, object]:
        out = [None] * self.world_size
        self._dist.all_gather_object(out, payload, group=self.pg)
        return dict(enumerate(out))

    def check(self, desc: tuple) -> None:
        """Optional ordering check (ref _checked_exchange): all ranks must issue
        the same collective descriptor."""
        if not self.check_order or self.world_size == 1:
            return
        digest = hashlib.sha1(repr(desc).encode()).hexdigest()
        got = self.exchange(self.rank, (digest, desc))
        if any(d != digest for d, _ in got.values()):
            raise RendezvousTimeout(f"collective mismatch across ranks (ordering bug): rank {self.rank} issued "
                                    f"{desc}, peers issued {sorted({repr(x) for _, x in got.values()})}")

    def agree(self, rank: int, src: int, value: object, tag: str = "") -> object:
        if self.world_size == 1:
            return value
        self.check(("agree", tag, src))
        box = [value if rank == src else None]
        self._dist.broadcast_object_list(box, src=self._global(src), group=self.pg,
                                         device=self.device if self.backend == "nccl" else None)
        return box[0]

    def abort(self, reason: str) -> None:
        raise RendezvousTimeout(reason)

    # -- data plane (raw tensors; the loader wraps them into TensorViews) ----------------
    def broadcast_tensor(self, t: torch.Tensor, src: int) -> None:
        """In-place broadcast of a contiguous tensor from group rank ``src``."""
        if self.world_size > 1 and t.numel():
            self._dist.broadcast(t, src=self._global(src), group=self.pg)

    def scatter_parts(self, rank: int, src: int, parts: list[torch.Tensor] | None, out: torch.Tensor) -> None:
        """Owner ``src`` sends ``parts[r]`` to every other rank r (its own part
        is already in ``out``); the others receive into ``out``. One grouped
        send/recv (ncclGroupStart/End under torch), so uneven remainder parts
        need no padding."""
        if self.world_size == 1:
            return
        ops = []
        if rank == src:
            if parts is None or len(parts) != self.world_size:
                raise SpecMismatch("scatter owner must provide one part per rank")
            ops = [("send", parts[r], r) for r in range(self.world_size) if r != src and parts[r].numel()]
        elif out.numel():
            ops = [("recv", out, src)]
        self.p2p(ops)

    def p2p(self, ops: list[tuple[str, torch.Tensor, int]]) -> None:
        """One grouped point-to-point call for a whole batch (ncclGroupStart /
        ncclGroupEnd under torch's batch_isend_irecv): ``ops`` are
        ("send" | "recv", contiguous tensor, group rank), posted in the same
        key order on every rank. gloo cannot move CUDA tensors point to point,
        so there they are staged through host memory."""
        if not ops or self.world_size == 1:
            return
        dist = self._dist
        stage = self.backend == "gloo"
        staged, posted = [], []
        for kind, t, peer in ops:
            h = t
            if stage and t.is_cuda:
                if kind == "send":
                    h = t.cpu()
                else:
                    h = torch.empty(t.shape, dtype=t.dtype)
                    staged.append((t, h))
            posted.append(dist.P2POp(dist.isend if kind == "send" else dist.irecv, h, self._global(peer), group=self.pg))
        for w in dist.batch_isend_irecv(posted):
            w.wait()
        for t, h in staged:
            t.copy_(h)

    # -- TensorView level (what the loader calls; same signatures as ProcessGroup) -------------
    def broadcast(self, rank: int, view, src: int, pool=None, tag: str = "", meta=None):
        """ncclBroadcast from ``src``; receivers allocate from their own pool.
        ``meta`` (every rank knows it from the headers) gives dtype and shape."""
        if not 0 <= src < self.world_size:
            raise ValueError(f"src {src} not in group of {self.world_size}")
        self.check(("broadcast", tag, src))
        if self.world_size == 1:
            if view is None:
                raise SpecMismatch("broadcast source holds no view")
            return view
        if rank == src:
            if view is None:
                raise SpecMismatch(f"broadcast src rank {src} holds no view (tag={tag!r})")
            self.broadcast_tensor(view.buffer.tensor[view.base_offset : view.base_offset + view.nbytes], src)
            return view
        if pool is None or meta is None:
            raise ValueError("non-source ranks need a destination pool and the tensor metadata")
        buf, out = _fresh(pool, tag or meta.name, meta.dtype, tuple(meta.shape))
        self.broadcast_tensor(buf.tensor[: out.nbytes], src)
        return out

    def scatter(self, rank: int, spec: ShardSpec, src: int, source_view=None, pool=None, tag: str = "",
                dtype: DType | None = None, src_dtype: DType | None = None):
        """Owner packs every rank's slice (cast fused) with ONE hl_gather launch
        — its own slice straight into its result — then one grouped NCCL
        send/recv delivers the rest. NVLink carries final-dtype bytes."""
        if spec.world_size != self.world_size:
            raise SpecMismatch(f"spec is for world {spec.world_size}, group is {self.world_size}")
        self.check(("scatter", tag, src, spec.dim, spec.full_shape))
        if self.world_size == 1:
            if source_view is None:
                raise SpecMismatch("scatter source holds no view")
            return source_view
        if pool is None:
            raise ValueError("scatter needs a destination pool on every rank")
        in_dtype = source_view.dtype if source_view is not None else src_dtype
        if in_dtype is None:
            raise ValueError("receivers must know the source dtype (src_dtype)")
        out_dtype = dtype or in_dtype
        buf, out = _fresh(pool, tag or spec.key, out_dtype, spec.part_shapes[rank])
        mine = buf.tensor[: out.nbytes]
        if rank != src:
            self.scatter_parts(rank, src, None, mine)
            return out
        if source_view is None:
            raise SpecMismatch(f"scatter src rank {src} holds no view (tag={tag!r})")
        if tuple(source_view.shape) != spec.full_shape:
            raise SpecMismatch(f"source shape {list(source_view.shape)} does not match spec {list(spec.full_shape)}")
        t = source_view.buffer.tensor
        parts = pack_parts(spec, source_view.buffer.ptr + source_view.base_offset, in_dtype, out_dtype,
                           own=src, own_out=mine, device=pool.device,
                           src_bytes=t[source_view.base_offset:source_view.base_offset + source_view.nbytes])
        self.scatter_parts(rank, src, parts, mine)
        return out
