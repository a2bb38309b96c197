"""TensorView parity with the reference's tests/test_tensorview.py: byte
strides (CPU), and on the GPU the zero-copy view, element decoding of every
dtype against the fixture bytes, scalar and zero-size views, release rules and
the JSON descriptor."""

from __future__ import annotations

import json
import math
import struct

import numpy as np
import pytest

from paper_2505_23072_b200.format import DType, TensorMetadata
from paper_2505_23072_b200.tensorview import compute_strides

gpu = pytest.mark.gpu


def meta(dtype, shape, begin=0, name="t"):
    nbytes = math.prod(shape) * dtype.size_bytes
    return TensorMetadata(name, dtype, tuple(shape), (begin, begin + nbytes))


# ----------------------------------------------------------------------- strides (CPU)
@pytest.mark.parametrize("shape,dtype,want", [((2, 3), DType.F32, (12, 4)), ((), DType.F16, ()),
                                              ((4, 1, 5), DType.I64, (40, 40, 8)), ((4, 0, 5), DType.U8, (0, 5, 1))])
def test_strides_known_answers(shape, dtype, want):
    """ref tests/test_tensorview.py:24-34."""
    assert compute_strides(shape, dtype) == want


def test_strides_are_row_major_contiguous(rng):
    for _ in range(200):
        shape = tuple(int(rng.integers(0, 6)) for _ in range(int(rng.integers(0, 5))))
        dtype = list(DType)[int(rng.integers(0, len(DType)))]
        s = compute_strides(shape, dtype)
        assert len(s) == len(shape)
        if shape:
            assert s[-1] == dtype.size_bytes
            assert all(s[i] == s[i + 1] * shape[i + 1] for i in range(len(shape) - 1))


# ----------------------------------------------------------------------- views (GPU)
@pytest.fixture
def pool():
    from paper_2505_23072_b200.device import DevicePool

    return DevicePool("host", device_id=0)


@gpu
def test_every_dtype_decodes_fixture_bytes(pool, rng):
    """Spot indices (corners + one random) of a random tensor of every dtype:
    read_element bits equal the fixture bytes; the torch alias and as_numpy
    hold the same bytes (ref tests/test_tensorview.py:126-150)."""
    from conftest import random_tensor_set

    from paper_2505_23072_b200.tensorview import make_view, read_element

    for dt in DType:
        for name, (dtype, shape, raw) in random_tensor_set(rng, 4, prefix=dt.value, dtypes=[dt]).items():
            buf = pool.allocate(max(len(raw), dtype.size_bytes))
            buf.write_bytes(0, raw)
            view = make_view(buf, 0, meta(dtype, shape, name=name))
            assert view.tobytes() == raw and view.as_numpy().tobytes() == raw
            assert tuple(view.torch.shape) == tuple(shape)
            if view.numel == 0:  # torch reports data_ptr 0 for empty tensors
                continue
            assert view.torch.data_ptr() == buf.ptr
            for flat in {0, view.numel - 1, int(rng.integers(0, view.numel))}:
                idx = tuple(int(i) for i in np.unravel_index(flat, shape)) if shape else ()
                start = flat * dtype.size_bytes
                assert read_element(view, idx).bits == int.from_bytes(raw[start:start + dtype.size_bytes], "little")


@gpu
def test_scalar_zero_size_and_index_errors(pool):
    from paper_2505_23072_b200.errors import IndexOutOfRange
    from paper_2505_23072_b200.tensorview import make_view, read_element

    buf = pool.allocate(32)
    buf.write_bytes(0, struct.pack("<d", 2.5) + np.arange(6, dtype=np.float32).tobytes())
    scalar = make_view(buf, 0, meta(DType.F64, ()))
    assert read_element(scalar, ()).value == 2.5 and scalar.torch.item() == 2.5 and scalar.strides == ()
    grid = make_view(buf, 8, meta(DType.F32, (2, 3)))
    assert read_element(grid, (1, 2)).value == 5.0 and read_element(grid, (0, 0)).value == 0.0
    for bad in [(2, 0), (0, 3), (0,), (0, 0, 0), (-1, 0)]:
        with pytest.raises(IndexOutOfRange):
            read_element(grid, bad)
    empty = make_view(buf, 32, meta(DType.U8, (4, 0, 5)))  # zero bytes at the very end is in bounds
    assert empty.numel == 0 and empty.tobytes() == b"" and empty.strides == (0, 5, 1)


@gpu
def test_live_view_blocks_release_then_use_after_close(pool):
    from paper_2505_23072_b200.errors import UseAfterClose
    from paper_2505_23072_b200.tensorview import make_view, read_element

    buf = pool.allocate(16)
    view = make_view(buf, 0, meta(DType.U8, (4,)))
    with pytest.raises(ValueError):
        buf.release()
    buf.release(force=True)
    for op in (view.tobytes, view.as_numpy, lambda: read_element(view, (0,))):
        with pytest.raises(UseAfterClose):
            op()
    with pytest.raises(UseAfterClose):
        make_view(buf, 0, meta(DType.U8, (4,)))


@gpu
def test_descriptor_is_json_ready(pool):
    """ref tests/test_tensorview.py:153-164 (device 0: the box has one GPU)."""
    from paper_2505_23072_b200.tensorview import make_view

    view = make_view(pool.allocate(64), 8, meta(DType.I16, (2, 4)))
    assert json.loads(json.dumps(view.descriptor())) == {"device_id": 0, "offset": 8, "dtype": "I16",
                                                         "shape": [2, 4], "strides": [8, 2]}
