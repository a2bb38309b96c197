"""The device sub-boundary (ref device.py:238-590): transfer_from_file,
align_and_convert, align_fix and convert_dtype on the B200 (native engine +
hl_gather), checked three ways:

* whole-buffer replay of 240 reference-made cases (tests/golden/device_cases.json,
  made by tests/golden/make_device_golden.py): same returned table or metadata,
  same sha256 of every buffer byte afterwards (padding and narrowed tails
  included), or the same error class;
* the reference's own known answers (ref tests/test_device.py:181-360): the
  repack targets of odd headers and mixed-direction movers, the direct
  backends' alignment rule, EOF;
* a conversion sweep of every supported pair against the numpy oracle table
  (tests/golden/conv.npz), in place.
"""

from __future__ import annotations

import base64
import hashlib
import json
import math
import struct

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import GOLDEN  # noqa: E402
from paper_2505_23072_b200.device import (  # noqa: E402
    DeviceBackend,
    DevicePool,
    align_and_convert,
    align_fix,
    convert_dtype,
    transfer_from_file,
)
from paper_2505_23072_b200.errors import (  # noqa: E402
    BounceTooSmall,
    IoError,
    MisalignedDirectTransfer,
    OutOfBoundsView,
    UnsupportedConversion,
)
from paper_2505_23072_b200.format import DType, TensorMetadata  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = json.loads((GOLDEN / "device_cases.json").read_text())["cases"]


def tmeta(name, dtype, shape, begin=0):
    nbytes = math.prod(shape) * dtype.size_bytes
    return TensorMetadata(name, dtype, tuple(shape), (begin, begin + nbytes))


def loaded(raw: bytes, backend="host"):
    buf = DevicePool(backend, device_id=0).allocate(len(raw))
    buf.write_bytes(0, raw)
    return buf


# ----------------------------------------------------------------------- reference replay
@pytest.mark.parametrize("i", range(len(CASES)))
def test_matches_reference_whole_buffer(i):
    c = CASES[i]
    raw = base64.b64decode(c["input"])
    buf = loaded(raw)
    exp = c["expect"]
    try:
        if c["op"] == "align_and_convert":
            landing = [(n, o, TensorMetadata(n, DType.from_tag(t), tuple(s), (0, math.prod(s) * DType.from_tag(t).size_bytes)))
                       for n, o, t, s in c["landing"]]
            table = align_and_convert(buf, landing, c["bounce"],
                                      {k: DType.from_tag(v) for k, v in c["conversions"].items()})
            got = {"table": [[n, o, m.dtype.value, list(m.data_offsets)] for n, o, m in table]}
        else:
            dt = DType.from_tag(c["dtype"])
            m = TensorMetadata("t", dt, (c["numel"],), (c["begin"], c["begin"] + c["numel"] * dt.size_bytes))
            out = convert_dtype(buf, m, DType.from_tag(c["target"]), c["bounce"])
            got = {"meta": [out.dtype.value, list(out.data_offsets)]}
        torch.cuda.synchronize()
        got["sha256"] = hashlib.sha256(buf.read_bytes(0, len(raw))).hexdigest()
    except Exception as e:  # noqa: BLE001 - the class name is the outcome
        got = {"error": type(e).__name__}
    assert got == exp, c
    if "error" in exp:  # a refused call leaves the buffer untouched
        assert buf.read_bytes(0, len(raw)) == raw


# ----------------------------------------------------------------------- known answers
def test_odd_header_single_tensor_compacts_to_zero(rng):
    """body at 107 (ref test_device.py:258): the F32 lands at 107 and moves to 0."""
    payload = rng.integers(0, 256, size=24, dtype=np.uint8).tobytes()
    buf = loaded(bytes(107) + payload)
    assert align_fix(buf, [("a0", 107, tmeta("a0", DType.F32, (2, 3)))], bounce=16) == [("a0", 0)]
    assert buf.read_bytes(0, 24) == payload


@pytest.mark.parametrize("layout,want", [
    ([("h", 3, DType.F16, 8), ("d", 19, DType.F64, 1)], {"h": 0, "d": 16}),
    ([("a", 2, DType.U8, 1), ("b", 3, DType.F64, 1)], {"a": 0, "b": 8}),            # right-moving F64
    ([("a", 2, DType.U8, 1), ("b", 3, DType.F64, 1), ("c", 11, DType.U8, 1)], {"a": 0, "b": 8, "c": 16}),
    ([("t", 107, DType.F32, 1000)], {"t": 0}),                                       # large shift
])
def test_repack_targets(rng, layout, want):
    cap = max(o + n * d.size_bytes for _, o, d, n in layout) + 16
    raw = bytearray(rng.integers(0, 256, size=cap, dtype=np.uint8).tobytes())
    buf = loaded(bytes(raw))
    landing = [(k, o, tmeta(k, d, (n,))) for k, o, d, n in layout]
    assert dict(align_fix(buf, landing, bounce=8)) == want
    for k, o, d, n in layout:
        assert buf.read_bytes(want[k], n * d.size_bytes) == bytes(raw[o:o + n * d.size_bytes]), k


def test_aligned_landing_is_noop_and_idempotent(rng):
    raw = rng.integers(0, 256, size=64, dtype=np.uint8).tobytes()
    buf = loaded(raw)
    landing = [("x", 8, tmeta("x", DType.F64, (3,))), ("y", 32, tmeta("y", DType.F32, (4,)))]
    assert align_fix(buf, landing, bounce=64) == [("x", 8), ("y", 32)]
    assert buf.read_bytes(0, 64) == raw
    buf2 = loaded(raw)
    table = align_fix(buf2, [("t", 5, tmeta("t", DType.F32, (6,)))], bounce=8)
    before = buf2.read_bytes(0, 64)
    assert align_fix(buf2, [(n, o, tmeta(n, DType.F32, (6,))) for n, o in table], bounce=8) == table
    assert buf2.read_bytes(0, 64) == before


def test_bounce_too_small_and_capacity():
    buf = loaded(bytes(64))
    with pytest.raises(BounceTooSmall):
        align_fix(buf, [("t", 3, tmeta("t", DType.F64, (2,)))], bounce=4)
    with pytest.raises(OutOfBoundsView):  # F16 -> F32 needs 32 bytes at 0; capacity 16
        convert_dtype(loaded(bytes(16)), tmeta("t", DType.F16, (8,)), DType.F32)
    with pytest.raises(UnsupportedConversion):
        convert_dtype(buf, tmeta("t", DType.F64, (1,)), DType.F16)


@pytest.mark.parametrize("src,bits,dst,want", [
    (DType.BF16, 0x3F80, DType.F16, 0x3C00),   # 1.0
    (DType.BF16, 0x7F80, DType.F16, 0x7C00),   # +inf
    (DType.F32, 0x00000000, DType.F16, 0x0000),
    (DType.F32, 0x7149F2CA, DType.F16, 0x7C00),  # 1e30 overflows to +inf
])
def test_convert_known_values(src, bits, dst, want):
    raw = struct.pack("<I" if src.size_bytes == 4 else "<H", bits)
    buf = loaded(raw + bytes(16))
    out = convert_dtype(buf, TensorMetadata("t", src, (1,), (0, len(raw))), dst, bounce=16)
    assert out.dtype is dst and out.data_offsets == (0, dst.size_bytes)
    assert buf.read_bytes(0, 2) == struct.pack("<H", want)


@pytest.mark.parametrize("src,dst", [("F16", "F32"), ("BF16", "F16"), ("BF16", "F32"), ("F32", "F16")])
def test_convert_in_place_matches_oracle_table(src, dst):
    """Every input of the conversion table (conv.npz, made by the reference's
    numpy casts) converted in place at an aligned begin: bit-exact."""
    table = np.load(GOLDEN / "conv.npz")
    x = table["f32_in"] if src == "F32" else table["all16"]
    y = table[f"{src.lower()}_{dst.lower()}"]
    s, d = DType.from_tag(src), DType.from_tag(dst)
    begin = 8
    raw = bytes(begin) + x.tobytes()
    buf = loaded(raw + bytes(max(0, x.size * d.size_bytes - x.nbytes) + 8))
    convert_dtype(buf, TensorMetadata("t", s, (x.size,), (begin, begin + x.nbytes)), d)
    torch.cuda.synchronize()
    assert buf.read_bytes(begin, y.nbytes) == y.tobytes()


def test_convert_during_repack(rng):
    bits = rng.integers(0, 2 ** 16, size=33, dtype=np.uint16)
    buf = loaded(bytes(43) + bits.astype("<u2").tobytes() + bytes(256))
    (name, off, m), = align_and_convert(buf, [("w", 43, tmeta("w", DType.BF16, (33,)))], bounce=16,
                                        conversions={"w": DType.F16})
    assert off == 0 and m.dtype is DType.F16 and m.data_offsets == (0, 66)
    got = np.frombuffer(buf.read_bytes(0, 66), dtype="<u2")
    f32 = (bits.astype(np.uint32) << 16).view(np.float32)
    with np.errstate(over="ignore"):
        assert np.array_equal(got, f32.astype(np.float16).view("<u2"))


# ----------------------------------------------------------------------- transfer_from_file
@pytest.fixture
def blob(tmp_path, rng):
    data = rng.integers(0, 256, size=4096, dtype=np.uint8).tobytes()
    p = tmp_path / "blob.bin"
    p.write_bytes(data)
    return p, data


def test_host_transfer_odd_offsets_fd_fileobj_and_path(blob):
    path, data = blob
    buf = DevicePool("host", device_id=0).allocate(64)
    with open(path, "rb") as f:
        transfer_from_file(buf, 7, f, 3, 5)                 # file object (the reference's call)
        transfer_from_file(buf, 20, f.fileno(), 100, 11)    # raw fd
    transfer_from_file(buf, 40, str(path), 4090, 6)         # a path (extension)
    assert buf.read_bytes(7, 5) == data[3:8]
    assert buf.read_bytes(20, 11) == data[100:111]
    assert buf.read_bytes(40, 6) == data[4090:]


def test_host_transfer_small_bounce_and_bounds(blob):
    path, data = blob
    buf = DevicePool(DeviceBackend.host(bounce_buffer_bytes=4096), device_id=0).allocate(4096)
    with open(path, "rb") as f:
        transfer_from_file(buf, 0, f, 0, 4096)
        assert buf.read_bytes(0, 4096) == data
        with pytest.raises(OutOfBoundsView):
            transfer_from_file(DevicePool("host", device_id=0).allocate(16), 8, f, 0, 16)
        with pytest.raises(IoError):
            transfer_from_file(buf, 0, f, 4000, 200)        # past end of file
        with pytest.raises(BounceTooSmall):
            transfer_from_file(buf, 0, f, 0, 16, staging=np.empty(0, np.uint8))


@pytest.mark.parametrize("backend,align", [("simdirect", 512), ("gds", 4096)])
def test_direct_transfer_alignment_rule(tmp_path, rng, backend, align):
    data = rng.integers(0, 256, size=3 * align + 188, dtype=np.uint8).tobytes()
    p = tmp_path / "d.bin"
    p.write_bytes(data)
    buf = DevicePool(backend, device_id=0).allocate(4 * align)
    with open(p, "rb") as f:
        transfer_from_file(buf, 0, f, align, align)
        assert buf.read_bytes(0, align) == data[align:2 * align]
        transfer_from_file(buf, align, f, 3 * align, 188)   # short tail that ends at EOF: allowed
        assert buf.read_bytes(align, 188) == data[3 * align:]
        for dev_off, file_off, n in [(0, 100, align), (64, align, align), (0, 0, 300)]:
            with pytest.raises(MisalignedDirectTransfer):
                transfer_from_file(buf, dev_off, f, file_off, n)
