"""Golden outcomes of the REFERENCE's header parser/validator on fuzzed
headers (build container only; the reference does not exist on the GPU box).
Re-run:  python tests/golden/make_format_golden.py

Cases: valid random layouts, structured corruptions of every field the
reference checks (format.py:143-292: length prefix, JSON syntax, duplicate
keys, __metadata__ types, dtype tags, shape/offset types and signs, missing
fields, overlaps, gaps, ranges past the body, begin > end, size mismatches),
and random byte/length mutations. For each: the reference's outcome of
parse_header + validate(file_size) — the error class name, or the parsed
(body_offset, metadata, [(name, dtype, shape, offsets)]) — written to
tests/golden/format_cases.json; tests/test_format.py replays them.
"""

from __future__ import annotations

import base64
import json
import struct
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

from aggload.format import parse_header, validate  # noqa: E402  (reference code, read-only import)

DTYPES = ["BOOL", "U8", "I8", "I16", "U16", "I32", "U32", "I64", "U64", "F16", "BF16", "F32", "F64"]
SIZE = dict(zip(DTYPES, [1, 1, 1, 2, 2, 4, 4, 8, 8, 2, 2, 4, 8]))


def outcome(blob: bytes, file_size: int):
    try:
        h = parse_header(blob)
        validate(h, file_size)
    except Exception as e:  # noqa: BLE001 - the class name IS the outcome
        return {"error": type(e).__name__}
    return {"body_offset": h.body_offset, "metadata": h.metadata,
            "tensors": [[m.name, m.dtype.value, list(m.shape), list(m.data_offsets)] for m in h.tensors.values()]}


def layout(rng, n):
    doc, cur = {}, 0
    for i in range(n):
        dt = DTYPES[int(rng.integers(0, len(DTYPES)))]
        shape = [int(x) for x in rng.integers(0, 5, size=int(rng.integers(0, 3)))]
        nb = int(np.prod(shape, dtype=np.int64)) * SIZE[dt] if shape else SIZE[dt]
        doc[f"t{i}"] = {"dtype": dt, "shape": shape, "data_offsets": [cur, cur + nb]}
        cur += nb
    return doc, cur


def blob_of(doc_bytes: bytes) -> bytes:
    return struct.pack("<Q", len(doc_bytes)) + doc_bytes


def main():
    rng = np.random.default_rng(20250523)
    cases = []

    def add(doc_bytes: bytes, body_len: int, tag: str, prefix: bytes | None = None):
        blob = prefix if prefix is not None else blob_of(doc_bytes)
        size = len(blob) + body_len
        cases.append({"tag": tag, "blob": base64.b64encode(blob).decode(), "file_size": size,
                      "expect": outcome(blob, size)})

    for i in range(60):  # valid layouts (some with metadata)
        doc, body = layout(rng, int(rng.integers(0, 6)))
        if i % 3 == 0:
            doc = {"__metadata__": {"format": "pt", "i": str(i)}, **doc}
        add(json.dumps(doc).encode(), body, "valid")
        add(json.dumps(doc).encode(), body + int(rng.integers(1, 64)), "valid-slack")

    def mutate(name, fn, n=12):
        for _ in range(n):
            doc, body = layout(rng, int(rng.integers(1, 5)))
            keys = list(doc)
            k = keys[int(rng.integers(0, len(keys)))]
            fn(doc, k)
            add(json.dumps(doc).encode(), body, name)

    mutate("bad-dtype", lambda d, k: d[k].__setitem__("dtype", ["Q8", "f32", "", "FP8", 5][int(rng.integers(0, 5))]))
    mutate("negative-shape", lambda d, k: d[k].__setitem__("shape", [2, -1]))
    mutate("bool-shape", lambda d, k: d[k].__setitem__("shape", [True, 2]))
    mutate("float-shape", lambda d, k: d[k].__setitem__("shape", [2.0]))
    mutate("shape-not-list", lambda d, k: d[k].__setitem__("shape", 4))
    mutate("missing-field", lambda d, k: d[k].pop(["dtype", "shape", "data_offsets"][int(rng.integers(0, 3))]))
    mutate("entry-not-object", lambda d, k: d.__setitem__(k, [1, 2]))
    mutate("offsets-len", lambda d, k: d[k].__setitem__("data_offsets", d[k]["data_offsets"][:1]))
    mutate("offsets-negative", lambda d, k: d[k].__setitem__("data_offsets", [-1, d[k]["data_offsets"][1]]))
    mutate("offsets-bool", lambda d, k: d[k].__setitem__("data_offsets", [False, d[k]["data_offsets"][1]]))
    mutate("begin-after-end", lambda d, k: d[k].__setitem__("data_offsets", [d[k]["data_offsets"][1] + 1, d[k]["data_offsets"][1]]))
    mutate("size-mismatch", lambda d, k: d[k].__setitem__("data_offsets", [d[k]["data_offsets"][0], d[k]["data_offsets"][1] + 1]))
    mutate("past-body", lambda d, k: d[k].__setitem__("data_offsets", [d[k]["data_offsets"][0] + 10**6, d[k]["data_offsets"][1] + 10**6]))
    mutate("metadata-nonstr", lambda d, k: d.__setitem__("__metadata__", {"a": 1}))
    mutate("metadata-notdict", lambda d, k: d.__setitem__("__metadata__", ["a"]))

    for _ in range(12):  # overlap: second tensor starts inside the first
        add(json.dumps({"a": {"dtype": "F32", "shape": [4], "data_offsets": [0, 16]},
                        "b": {"dtype": "U8", "shape": [8], "data_offsets": [8, 16]}}).encode(), 16, "overlap")
    for gap in (1, 7, 64):  # gaps are legal
        add(json.dumps({"a": {"dtype": "F32", "shape": [4], "data_offsets": [0, 16]},
                        "b": {"dtype": "U8", "shape": [8], "data_offsets": [16 + gap, 24 + gap]}}).encode(),
            24 + gap, "gap")
    add(b'{"a":{"dtype":"U8","shape":[1],"data_offsets":[0,1]},"a":{"dtype":"U8","shape":[1],"data_offsets":[1,2]}}',
        2, "duplicate-key")
    add(b"{not json}", 0, "bad-json")
    add(b"[1,2]", 0, "json-not-object")
    add(b"", 0, "empty-doc")
    add(b"{}", 0, "empty-layout")
    add(b"{}", 0, "short-prefix", prefix=b"\x05\x00\x00")
    add(b"{}", 0, "declared-longer", prefix=struct.pack("<Q", 64) + b"{}")
    add(b"{}", 0, "huge-length", prefix=struct.pack("<Q", 2**40) + b"{}")
    add(json.dumps({"s": {"dtype": "F32", "shape": [], "data_offsets": [0, 4]}}).encode(), 4, "scalar")
    add(json.dumps({"z": {"dtype": "F32", "shape": [0, 3], "data_offsets": [5, 5]}}).encode(), 8, "zero-size")
    add(json.dumps({"t": {"dtype": "U8", "shape": [4], "data_offsets": [0, 4]}}).encode(), 2, "body-short")

    for _ in range(60):  # random byte flips in valid blobs
        doc, body = layout(rng, int(rng.integers(1, 4)))
        raw = bytearray(blob_of(json.dumps(doc).encode()))
        for _ in range(int(rng.integers(1, 4))):
            raw[int(rng.integers(0, len(raw)))] = int(rng.integers(0, 256))
        blob = bytes(raw)
        cases.append({"tag": "byte-flip", "blob": base64.b64encode(blob).decode(), "file_size": len(blob) + body,
                      "expect": outcome(blob, len(blob) + body)})

    (HERE / "format_cases.json").write_text(json.dumps({"cases": cases}, indent=0) + "\n")
    kinds = {}
    for c in cases:
        k = c["expect"].get("error", "ok")
        kinds[k] = kinds.get(k, 0) + 1
    print(f"wrote {len(cases)} cases: {kinds}")


if __name__ == "__main__":
    main()
