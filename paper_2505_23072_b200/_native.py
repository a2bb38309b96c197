"""ctypes binding of libhbmload.so (the C ABI in include/hbmload.h).

The library is built in-tree (``paper_2505_23072_b200/libhbmload.so``) by
``__graft_entry__.build()`` / ``python -m paper_2505_23072_b200._build``.
ctypes releases the GIL for the duration of every foreign call, so the
I/O engine's blocking ``hl_execute_plan`` never stalls other Python threads
(e.g. thread ranks of an in-process group).

There is no fallback: if the library is missing, every entry point raises
:class:`~paper_2505_23072_b200.errors.NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import struct
import threading
from pathlib import Path

from .errors import NativeUnavailable, raise_native

LIB_PATH = Path(__file__).resolve().parent / "libhbmload.so"

HL_IO_AUTO, HL_IO_BUFFERED, HL_IO_DIRECT, HL_IO_CUFILE, HL_IO_MMAP = 0, 1, 2, 3, 4
IO_MODE_NAMES = {HL_IO_BUFFERED: "buffered", HL_IO_DIRECT: "direct", HL_IO_CUFILE: "cufile", HL_IO_MMAP: "mmap",
                 5: "io_uring"}  # 5: HL_IO_USED_URING (hbmload.h)
IO_MODES = {"auto": HL_IO_AUTO, "buffered": HL_IO_BUFFERED, "direct": HL_IO_DIRECT, "cufile": HL_IO_CUFILE,
            "mmap": HL_IO_MMAP}


class hl_config(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("workers", C.c_uint32),
        ("chunk_bytes", C.c_uint64),
        ("slots_per_worker", C.c_uint32),
        ("io_mode", C.c_uint32),
        ("numa_node", C.c_int32),
        ("flags", C.c_uint32),
    ]


HL_CFG_AUTO_PIN_CACHE = 1


class hl_block(C.Structure):
    _fields_ = [
        ("file", C.c_uint32),
        ("worker", C.c_uint32),
        ("file_off", C.c_uint64),
        ("len", C.c_uint64),
        ("dev_dst", C.c_uint64),
    ]


class hl_plan_stats(C.Structure):
    _fields_ = [
        ("bytes", C.c_uint64),
        ("seconds", C.c_double),
        ("workers", C.c_uint32),
        ("blocks", C.c_uint32),
        ("direct_bytes", C.c_uint64),
        ("buffered_bytes", C.c_uint64),
        ("cufile_bytes", C.c_uint64),
        ("mmap_bytes", C.c_uint64),
        ("ring_setup_seconds", C.c_double),
        ("io_mode_used", C.c_uint32),
        ("numa_node", C.c_int32),
        ("read_seconds", C.c_double),
        ("wait_seconds", C.c_double),
        ("submit_seconds", C.c_double),
        ("setup_seconds", C.c_double),
        ("first_h2d_seconds", C.c_double),
        ("last_h2d_seconds", C.c_double),
    ]


class hl_desc(C.Structure):
    _fields_ = [
        ("src", C.c_uint64),
        ("dst", C.c_uint64),
        ("rows", C.c_uint64),
        ("row_elems", C.c_uint64),
        ("src_pitch", C.c_uint64),
        ("src_dtype", C.c_uint32),
        ("dst_dtype", C.c_uint32),
    ]


class hl_ipc_handle(C.Structure):
    _fields_ = [("handle", C.c_uint8 * 64), ("offset", C.c_uint64)]


# name -> (restype, argtypes): every symbol include/hbmload.h declares
SIGNATURES = {
    "hl_version": (C.c_char_p, []),
    "hl_last_error": (C.c_char_p, []),
    "hl_abi_version": (C.c_int, []),
    "hl_ctx_create": (C.c_int, [C.POINTER(hl_config), C.POINTER(C.c_void_p)]),
    "hl_ctx_destroy": (C.c_int, [C.c_void_p]),
    "hl_ctx_config": (C.c_int, [C.c_void_p, C.POINTER(hl_config)]),
    "hl_execute_plan": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p), C.c_uint32,
                                  C.POINTER(hl_block), C.c_uint32, C.POINTER(hl_plan_stats)]),
    "hl_execute_plan_after": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p), C.c_uint32,
                                        C.POINTER(hl_block), C.c_uint32, C.c_void_p, C.POINTER(hl_plan_stats)]),
    "hl_execute_plan_async": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p), C.c_uint32,
                                        C.POINTER(hl_block), C.c_uint32, C.c_void_p, C.POINTER(hl_plan_stats)]),
    "hl_ctx_cpus": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_uint32, C.POINTER(C.c_uint32)]),
    "hl_storage_numa_node": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32)]),
    "hl_topology_resolve": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.c_uint32, C.POINTER(C.c_uint32)]),
    "hl_transfer_from_file": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.c_uint64, C.c_void_p]),
    "hl_file_residency": (C.c_int, [C.c_char_p, C.POINTER(C.c_double)]),
    "hl_drop_cache": (C.c_int, [C.c_char_p]),
    "hl_gds_available": (C.c_int, []),
    "hl_conversion_supported": (C.c_int, [C.c_uint32, C.c_uint32]),
    "hl_gather": (C.c_int, [C.POINTER(hl_desc), C.c_uint32, C.c_void_p]),
    "hl_gather_ex": (C.c_int, [C.POINTER(hl_desc), C.c_uint32, C.c_void_p, C.c_uint32]),
    "hl_ipc_export": (C.c_int, [C.c_void_p, C.POINTER(hl_ipc_handle)]),
    "hl_ipc_import": (C.c_int, [C.POINTER(hl_ipc_handle), C.c_int, C.POINTER(C.c_void_p)]),
    "hl_ipc_release": (C.c_int, [C.c_void_p]),
    "hl_enable_peer_access": (C.c_int, [C.c_int, C.c_int]),
    "hl_gather_max_batch": (C.c_uint32, []),
    "hl_kernel_launches": (C.c_uint64, []),
    "hl_gather_timing": (C.c_int, [C.c_int]),
    "hl_gather_timings": (C.c_int, [C.POINTER(C.c_float), C.c_uint32, C.POINTER(C.c_uint32)]),
    "hl_gather_prepare": (C.c_int, [C.c_int]),
}

_lib = None
_lock = threading.Lock()


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the CDLL with typed signatures."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else Path(os.environ.get("HL_LIB", LIB_PATH))  # HL_LIB: tuning builds
        if not p.exists():
            raise NativeUnavailable(
                f"{p} is missing: build it with `python -m paper_2505_23072_b200._build` "
                "(there is no CPU fallback for the load path)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.hl_last_error().decode(errors="replace") if _lib is not None else ""
        raise_native(rc, msg or f"native call failed with status {rc}")


def conversion_supported(src_code: int, dst_code: int) -> bool:
    return bool(load().hl_conversion_supported(src_code, dst_code))


def kernel_launches() -> int:
    return int(load().hl_kernel_launches())


def gather_timing(enable: bool) -> None:
    """Switch hl_gather's launch timing (events around each call's kernel launches)."""
    check(load().hl_gather_timing(1 if enable else 0))


def gather_timings() -> list[float]:
    """Milliseconds of every hl_gather call recorded since the last fetch, in call order
    (waits for them to finish)."""
    lib = load()
    n = C.c_uint32()
    cap = 4096
    arr = (C.c_float * cap)()
    check(lib.hl_gather_timings(arr, cap, C.byref(n)))
    return [float(arr[i]) for i in range(min(n.value, cap))]


_prepared: set[int] = set()


def gather_prepare(device: int) -> None:
    """Load the hl_gather kernels for ``device`` ahead of their first launch
    (once per process; ctypes drops the GIL, so this overlaps a transfer)."""
    if device in _prepared:
        return
    check(load().hl_gather_prepare(device))
    _prepared.add(device)


_DESC = struct.Struct("<5Q2I")  # hl_desc, include/hbmload.h (48 bytes, no padding)
assert _DESC.size == C.sizeof(hl_desc)


def pack(descs: list[tuple]):
    """The descriptor table for ``hl_gather``: one struct.pack per entry into
    a single buffer (~3x cheaper than building ctypes Structures: this runs on
    the host before the launch, while the GPU waits)."""
    if len(descs) == 1:
        return C.byref(hl_desc(*descs[0])), 1
    return (hl_desc * len(descs)).from_buffer_copy(b"".join([_DESC.pack(*d) for d in descs])), len(descs)


GATHER_NO_TMA = 1  # include/hbmload.h HL_GATHER_NO_TMA


def launch(table, n: int, stream_ptr: int, flags: int = 0) -> None:
    lib = _lib or load()
    if flags:
        check(lib.hl_gather_ex(table, n, C.c_void_p(stream_ptr), flags))
    else:
        check(lib.hl_gather(table, n, C.c_void_p(stream_ptr)))


def gather(descs: list[tuple], stream_ptr: int, flags: int = 0) -> None:
    """Enqueue ``[(src, dst, rows, row_elems, src_pitch, src_code, dst_code), ...]``."""
    if descs:
        launch(*pack(descs), stream_ptr, flags)


class IoEngine:
    """One hl_ctx: worker threads' pinned ring + streams for one device."""

    def __init__(self, device: int, workers: int = 0, chunk_bytes: int = 0,
                 slots_per_worker: int = 0, io_mode: str = "auto", numa_node: int = -1, flags: int = 0):
        lib = load()
        cfg = hl_config(device, workers, chunk_bytes, slots_per_worker, IO_MODES[io_mode], numa_node, flags)
        h = C.c_void_p()
        check(lib.hl_ctx_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._lib = lib
        eff = hl_config()
        check(lib.hl_ctx_config(h, C.byref(eff)))
        self.config = {f: getattr(eff, f) for f, _ in hl_config._fields_}

    def execute(self, paths: list[str], blocks: list[tuple[int, int, int, int, int]],
                after_stream: int | None = None, async_tail: bool = False) -> dict:
        """blocks: (file_index, worker_hint, file_off, len, dev_dst). Blocking.
        ``after_stream`` (a cudaStream_t as int, 0 = legacy default): the
        engine's HBM writes wait for everything already queued on it
        (hl_execute_plan_after); None = unordered (hl_execute_plan).
        ``async_tail``: return once every copy is submitted, with the stream
        waiting for their completion (hl_execute_plan_async)."""
        lib = self._lib
        cpaths = (C.c_char_p * len(paths))(*[os.fsencode(p) for p in paths])
        arr = (hl_block * len(blocks))(*[hl_block(*b) for b in blocks])
        st = hl_plan_stats()
        if after_stream is None:
            check(lib.hl_execute_plan(self._h, cpaths, len(paths), arr, len(blocks), C.byref(st)))
        else:
            fn = lib.hl_execute_plan_async if async_tail else lib.hl_execute_plan_after
            check(fn(self._h, cpaths, len(paths), arr, len(blocks), C.c_void_p(after_stream), C.byref(st)))
        modes = [name for bit, name in IO_MODE_NAMES.items() if st.io_mode_used & (1 << bit)]
        return {
            "bytes": st.bytes, "seconds": st.seconds, "workers": st.workers, "blocks": st.blocks,
            "direct_bytes": st.direct_bytes, "buffered_bytes": st.buffered_bytes,
            "cufile_bytes": st.cufile_bytes, "mmap_bytes": st.mmap_bytes,
            "ring_setup_seconds": st.ring_setup_seconds,
            "read_seconds": st.read_seconds, "wait_seconds": st.wait_seconds,
            "submit_seconds": st.submit_seconds, "setup_seconds": st.setup_seconds,
            "first_h2d_seconds": st.first_h2d_seconds, "last_h2d_seconds": st.last_h2d_seconds,
            "io_modes": modes, "numa_node": st.numa_node,
        }

    def cpus(self) -> list[int]:
        """CPUs the worker team and the pinned ring are bound to ([] = unpinned)."""
        n = C.c_uint32()
        check(self._lib.hl_ctx_cpus(self._h, None, 0, C.byref(n)))
        arr = (C.c_int32 * max(n.value, 1))()
        check(self._lib.hl_ctx_cpus(self._h, arr, n.value, C.byref(n)))
        return list(arr[:n.value])

    def transfer(self, path: str, file_off: int, length: int, dev_ptr: int, after_stream: int = 0) -> None:
        """One range, ordered after ``after_stream`` (hl_execute_plan_after)."""
        if length:
            self.execute([path], [(0, 0, file_off, length, dev_ptr)], after_stream=after_stream)

    def close(self) -> None:
        if self._h:
            self._lib.hl_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def topology_resolve(pci_bus_id: str = "", requested_node: int = -1) -> tuple[int, list[int]]:
    """The engine's placement rule without a GPU (hl_topology_resolve):
    (NUMA node, CPUs the workers would be pinned to)."""
    lib = load()
    node, n = C.c_int32(), C.c_uint32()
    check(lib.hl_topology_resolve(pci_bus_id.encode(), requested_node, C.byref(node), None, 0, C.byref(n)))
    arr = (C.c_int32 * max(n.value, 1))()
    check(lib.hl_topology_resolve(pci_bus_id.encode(), requested_node, C.byref(node), arr, n.value, C.byref(n)))
    return node.value, list(arr[:n.value])


def storage_numa_node(path: str) -> int:
    """NUMA node of the storage device holding ``path`` (hl_storage_numa_node), -1 if unknown."""
    node = C.c_int32()
    check(load().hl_storage_numa_node(str(path).encode(), C.byref(node)))
    return node.value


def file_residency(path: str) -> float:
    lib = load()
    f = C.c_double()
    check(lib.hl_file_residency(os.fsencode(path), C.byref(f)))
    return f.value


def drop_cache(path: str) -> None:
    check(load().hl_drop_cache(os.fsencode(path)))


def gds_available() -> bool:
    return bool(load().hl_gds_available())


def ipc_export(dev_ptr: int) -> tuple[bytes, int]:
    """(handle bytes, offset) of the allocation holding ``dev_ptr``: picklable."""
    h = hl_ipc_handle()
    check(load().hl_ipc_export(C.c_void_p(dev_ptr), C.byref(h)))
    return bytes(h.handle), int(h.offset)


def ipc_import(handle: tuple[bytes, int], device: int) -> int:
    h = hl_ipc_handle()
    C.memmove(h.handle, handle[0], 64)
    h.offset = handle[1]
    out = C.c_void_p()
    check(load().hl_ipc_import(C.byref(h), device, C.byref(out)))
    return int(out.value)


def ipc_release(ptr: int) -> None:
    check(load().hl_ipc_release(C.c_void_p(ptr)))


_peer_enabled: set[tuple[int, int]] = set()


def enable_peer_access(device: int, peer: int) -> None:
    if device == peer or (device, peer) in _peer_enabled:
        return
    check(load().hl_enable_peer_access(device, peer))
    _peer_enabled.add((device, peer))
