"""safetensors parsing/validation/writing (CPU; ref pkg/tests/test_format.py behaviours)."""

from __future__ import annotations

import json
import struct

import numpy as np
import pytest

from conftest import GOLDEN, random_tensor_set
from oracle import oracle
from paper_2505_23072_b200.errors import (
    HeaderTooLarge,
    LengthMismatch,
    MalformedJson,
    NegativeShape,
    OffsetOutOfBounds,
    OverlappingTensors,
    SizeMismatch,
    TruncatedHeader,
    UnknownDType,
)
from paper_2505_23072_b200.format import DType, parse_header, read_header, validate, write_file, write_file_stream


def _blob(layout: dict, body: bytes = b"") -> bytes:
    doc = json.dumps(layout).encode()
    return struct.pack("<Q", len(doc)) + doc + body


def test_empty_layout():
    h = parse_header(struct.pack("<Q", 2) + b"{}")
    assert h.header_len == 2 and h.tensors == {} and h.body_offset == 10


def test_round_trip_random(rng):
    for trial in range(30):
        t = random_tensor_set(rng, int(rng.integers(0, 8)), prefix=f"r{trial}_")
        meta = {"format": "pt"} if trial % 2 else None
        blob = write_file(t, metadata=meta)
        h = parse_header(blob)
        validate(h, len(blob))
        assert h.metadata == meta
        for k, (dt, shape, raw) in t.items():
            m = h.tensors[k]
            assert m.dtype is dt and m.shape == shape and m.nbytes == len(raw)
            assert blob[h.body_offset + m.begin: h.body_offset + m.end] == raw


def test_pad_header_to_gives_odd_body():
    blob = write_file({"a0": (DType.F32, (2, 3), bytes(24))}, pad_header_to=99)
    assert parse_header(blob).body_offset == 107


def test_errors():
    with pytest.raises(TruncatedHeader):
        parse_header(b"\x01\x00")
    with pytest.raises(HeaderTooLarge):
        parse_header(struct.pack("<Q", 10**9), header_cap=10**8)
    with pytest.raises(TruncatedHeader):
        parse_header(struct.pack("<Q", 50) + b"{}")
    with pytest.raises(MalformedJson):
        parse_header(struct.pack("<Q", 3) + b"{x}")
    with pytest.raises(MalformedJson):
        doc = b'{"a":1,"a":2}'
        parse_header(struct.pack("<Q", len(doc)) + doc)
    with pytest.raises(UnknownDType):
        parse_header(_blob({"t": {"dtype": "Q8", "shape": [1], "data_offsets": [0, 1]}}))
    with pytest.raises(NegativeShape):
        parse_header(_blob({"t": {"dtype": "U8", "shape": [-1], "data_offsets": [0, 1]}}))
    with pytest.raises(MalformedJson):
        parse_header(_blob({"t": {"dtype": "U8", "shape": [True], "data_offsets": [0, 1]}}))
    with pytest.raises(MalformedJson):
        parse_header(_blob({"__metadata__": {"k": 1}}))
    with pytest.raises(LengthMismatch):
        write_file({"t": (DType.F32, (2,), bytes(7))})


def test_validate():
    ok = _blob({"t": {"dtype": "F32", "shape": [2, 3], "data_offsets": [0, 24]}}, bytes(24))
    validate(parse_header(ok), len(ok))
    bad = _blob({"t": {"dtype": "F32", "shape": [2, 3], "data_offsets": [0, 20]}}, bytes(24))
    with pytest.raises(SizeMismatch):
        validate(parse_header(bad), len(bad))
    ov = _blob({"a": {"dtype": "U8", "shape": [24], "data_offsets": [0, 24]},
                "b": {"dtype": "U8", "shape": [24], "data_offsets": [16, 40]}}, bytes(40))
    with pytest.raises(OverlappingTensors):
        validate(parse_header(ov), len(ov))
    past = _blob({"a": {"dtype": "U8", "shape": [24], "data_offsets": [0, 24]}}, bytes(10))
    with pytest.raises(OffsetOutOfBounds):
        validate(parse_header(past), len(past))
    gap = _blob({"a": {"dtype": "U8", "shape": [4], "data_offsets": [8, 12]}}, bytes(16))
    validate(parse_header(gap), len(gap))  # gaps are legal


def test_length_field_mutations_never_crash():
    blob = write_file({"t": (DType.U8, (4,), b"abcd")})
    for i in range(8):
        for v in (0, 1, 0x7F, 0xFF):
            b = bytearray(blob)
            b[i] = v
            try:
                h = parse_header(bytes(b))
                validate(h, len(b))
            except (TruncatedHeader, HeaderTooLarge, MalformedJson, OffsetOutOfBounds, SizeMismatch):
                pass


def test_golden_corpora_parse_like_the_oracle():
    for p in sorted((GOLDEN / "corpora").glob("*.safetensors")):
        h = read_header(p)
        validate(h, h.file_size)
        body, tensors = oracle.read_header(p)
        assert h.body_offset == body
        assert {k: (m.dtype.value, m.shape, m.begin, m.end) for k, m in h.tensors.items()} == tensors


def test_stream_writer(tmp_path):
    ents = [("a", DType.F32, (3,)), ("b", DType.U8, (5,))]
    data = [np.arange(3, dtype=np.float32), np.arange(5, dtype=np.uint8)]
    h = write_file_stream(tmp_path / "s.safetensors", ents, lambda i: data[i])
    assert h.body_offset % 8 == 0
    got = oracle.load_all([tmp_path / "s.safetensors"])
    assert got["a"][1] == data[0].tobytes() and got["b"][1] == data[1].tobytes()


def test_reference_outcomes_on_fuzzed_headers():
    """386 headers (valid layouts, every field corruption the reference checks,
    random byte flips) give the SAME outcome as the reference's parse_header +
    validate: the same error class, or the same parsed layout
    (tests/golden/format_cases.json, made by the reference itself)."""
    import base64

    from paper_2505_23072_b200 import errors

    cases = json.loads((GOLDEN / "format_cases.json").read_text())["cases"]
    mismatches = []
    for c in cases:
        blob = base64.b64decode(c["blob"])
        try:
            h = parse_header(blob)
            validate(h, c["file_size"])
            got = {"body_offset": h.body_offset, "metadata": h.metadata,
                   "tensors": [[m.name, m.dtype.value, list(m.shape), list(m.data_offsets)] for m in h.tensors.values()]}
        except errors.AggloadError as e:
            got = {"error": type(e).__name__}
        if got != c["expect"]:
            mismatches.append((c["tag"], c["expect"], got))
    assert not mismatches, mismatches[:5]


def test_entry_fast_path_matches_the_full_checker():
    """format._entry_fast (the well-formed-header shortcut) returns what
    format._entry returns and raises what it raises, over random entries:
    valid ones and every kind of malformed field (wrong types, bools as
    ints, negative dims/offsets, unknown dtypes, missing or extra keys)."""
    import random

    from paper_2505_23072_b200 import format as F

    rng = random.Random(5)
    tags = [d.value for d in F.DType] + ["F8", "bf16", 3, None]

    def val(kind):
        return rng.choice({
            "int": [0, 1, 7, 4096, -1, True, False, 2.0, "3", None],
            "list": [[], [1, 2], [0], [3, -1], [True, 2], [1.0], "12", None, [1, [2]]],
        }[kind])

    for _ in range(4000):
        e = {}
        if rng.random() < 0.95:
            e["dtype"] = rng.choice(tags)
        if rng.random() < 0.95:
            e["shape"] = val("list") if rng.random() < 0.3 else [rng.randint(0, 9) for _ in range(rng.randint(0, 3))]
        if rng.random() < 0.95:
            e["data_offsets"] = val("list") if rng.random() < 0.3 else [rng.randint(0, 99), rng.randint(0, 99)]
        if rng.random() < 0.1:
            e["extra"] = 1
        obj = e if rng.random() < 0.97 else rng.choice([[1], "x", 3])

        def run(fn):
            try:
                return ("ok", fn("t", obj))
            except Exception as ex:  # noqa: BLE001 - compared by class and message
                return ("err", type(ex).__name__, str(ex))

        assert run(F._entry_fast) == run(F._entry), obj
