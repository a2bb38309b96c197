"""DevicePool / DeviceBuffer / TensorView semantics on HBM (ref pkg/tests/test_device.py
TestPool, pkg/tests/test_tensorview.py): accounting counters, exact-size reuse,
capacity cap, double release, live views blocking release, view construction
errors, strides and element decoding."""

from __future__ import annotations

import struct

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2505_23072_b200.device import DevicePool  # noqa: E402
from paper_2505_23072_b200.errors import (  # noqa: E402
    DoubleRelease,
    IndexOutOfRange,
    MisalignedView,
    OutOfBoundsView,
    OutOfMemory,
    UseAfterClose,
)
from paper_2505_23072_b200.format import DType, TensorMetadata  # noqa: E402
from paper_2505_23072_b200.tensorview import compute_strides, make_view, read_element  # noqa: E402

pytestmark = pytest.mark.gpu


def meta(dt, shape, begin=0):
    n = int(np.prod(shape)) * dt.size_bytes if shape else dt.size_bytes
    return TensorMetadata("t", dt, tuple(shape), (begin, begin + n))


def test_pool_accounting_and_reuse():
    pool = DevicePool("host")
    b = pool.allocate(1024, zero=True)
    assert b.capacity == 1024 and b.read_bytes(0, 1024) == bytes(1024) and pool.allocated_bytes == 1024
    b.release()
    assert pool.pooled_bytes == 1024 and pool.allocated_bytes == 0 and pool.cumulative_pooled_bytes == 1024
    c = pool.allocate(1024)  # exact-size reuse comes out of the pool
    assert pool.pooled_bytes == 0 and pool.allocated_bytes == 1024
    with pytest.raises(DoubleRelease):
        b.release()
    c.release(force=True, to_pool=False)
    assert pool.pooled_bytes == 0 and pool.allocated_bytes == 0


def test_capacity_cap_and_eviction():
    pool = DevicePool("host", capacity_cap=1 << 20)
    with pytest.raises(OutOfMemory):
        pool.allocate(2 << 20)
    a = pool.allocate(600 << 10)
    a.release()
    b = pool.allocate(700 << 10)  # pooled block evicted to make room
    assert pool.pooled_bytes == 0 and b.capacity == 700 << 10


def test_refcount_and_live_views_block_unforced_release():
    pool = DevicePool("host")
    b = pool.allocate(64)
    b.refcount = 1
    with pytest.raises(ValueError):
        b.release()
    b.refcount = 0
    v = make_view(b, 0, meta(DType.U8, (4,)))
    with pytest.raises(ValueError):
        b.release()
    b.release(force=True)
    with pytest.raises(UseAfterClose):
        v.tobytes()


def test_views_alias_without_copy_and_errors():
    pool = DevicePool("host")
    b = pool.allocate(64)
    b.write_bytes(0, bytes(range(24)))
    before = pool.allocated_bytes
    views = [make_view(b, 0, meta(DType.F32, (2, 3))) for _ in range(5)]
    assert pool.allocated_bytes == before and views[0].strides == (12, 4)
    assert views[0].torch.data_ptr() == b.ptr and views[0].tobytes() == bytes(range(24))
    with pytest.raises(MisalignedView):
        make_view(b, 2, meta(DType.F32, (2,)))
    with pytest.raises(OutOfBoundsView):
        make_view(b, 56, meta(DType.F32, (4,)))


def test_strides_match_reference_known_answers():
    # ref pkg/tests/test_tensorview.py:24-38
    assert compute_strides((2, 3), DType.F32) == (12, 4)
    assert compute_strides((), DType.F16) == ()
    assert compute_strides((4, 1, 5), DType.I64) == (40, 40, 8)
    assert compute_strides((4, 0, 5), DType.U8) == (0, 5, 1)


@pytest.mark.parametrize("dt,val,fmt", [(DType.F32, -2.5, "<f"), (DType.I16, -7, "<h"), (DType.F64, 3.25, "<d"),
                                        (DType.U64, 2**63 + 5, "<Q"), (DType.F16, 0.5, "<e")])
def test_read_element_decodes(dt, val, fmt):
    pool = DevicePool("host")
    b = pool.allocate(64)
    raw = struct.pack(fmt, val) * 3
    b.write_bytes(0, raw)
    v = make_view(b, 0, meta(dt, (3,)))
    e = read_element(v, (1,))
    assert e.value == float(val) and e.bits == int.from_bytes(struct.pack(fmt, val), "little")
    with pytest.raises(IndexOutOfRange):
        read_element(v, (3,))


def test_bf16_and_bool_surface_as_raw_bits():
    pool = DevicePool("host")
    b = pool.allocate(16)
    b.write_bytes(0, struct.pack("<HH", 0x3F80, 0xC000) + b"\x01\x00")
    bf = make_view(b, 0, meta(DType.BF16, (2,)))
    assert bf.as_numpy().tolist() == [0x3F80, 0xC000] and read_element(bf, (0,)).value == 1.0
    assert bf.torch.tolist() == [1.0, -2.0]
    bl = make_view(b, 4, meta(DType.BOOL, (2,)))
    assert bl.torch.tolist() == [True, False] and bl.as_numpy().tolist() == [1, 0]
