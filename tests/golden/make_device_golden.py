"""Golden whole-buffer traces of the REFERENCE device sub-boundary (build
container only; the reference does not exist on the GPU box). Re-run:
    python tests/golden/make_device_golden.py   -> tests/golden/device_cases.json

Each case is a small buffer of random bytes with tensors landed at random
(often misaligned, tightly packed) offsets, then ONE reference call:

  align_and_convert(buf, landing, bounce, conversions)   (ref device.py:466)
  convert_dtype(buf, meta, target, bounce)               (ref device.py:551)

Recorded: the input bytes (base64), the arguments, and either the returned
table plus the sha256 of the WHOLE buffer afterwards (padding and tails
included) or the error class. tests/test_device_ops_gpu.py replays every case
on the B200 implementation (paper_2505_23072_b200.device) and demands the same.
"""

from __future__ import annotations

import base64
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

from aggload.device import DevicePool, align_and_convert, convert_dtype  # noqa: E402  (read-only import)
from aggload.format import DType, TensorMetadata  # noqa: E402

TAGS = ["U8", "I8", "BOOL", "F16", "BF16", "I16", "F32", "I32", "F64", "I64"]
CONV = {"F32": ["F16"], "F16": ["F32"], "BF16": ["F16", "F32"]}
SPECIAL = [0x0000, 0x8000, 0x7F80, 0xFF80, 0x7FC0, 0x7F81, 0xFFFF, 0x0001, 0x3F80, 0x477F, 0x4780]


def fill(rng, dtype, n):
    """Random bytes, salted with special bit patterns for the float dtypes."""
    raw = rng.integers(0, 256, size=n * dtype.size_bytes, dtype=np.uint8)
    if dtype.value in ("BF16", "F16") and n:
        v = raw.view("<u2").copy()
        pick = rng.random(n) < 0.3
        v[pick] = rng.choice(SPECIAL, size=int(pick.sum()))
        raw = v.view(np.uint8)
    if dtype.value == "F32" and n:
        v = raw.view("<u4").copy()
        pick = rng.random(n) < 0.3
        v[pick] = rng.choice([0x7F800000, 0xFF800000, 0x7FC00001, 0x7F800001, 0x477FF000, 0x47800000,
                              0x33800000, 0x387FC000, 0x00000001, 0x80000000], size=int(pick.sum()))
        raw = v.view(np.uint8)
    return raw.tobytes()


def repack_case(rng):
    n = int(rng.integers(1, 6))
    off = int(rng.integers(0, 9))
    tensors, landing, conversions = {}, [], {}
    for i in range(n):
        tag = TAGS[int(rng.integers(0, len(TAGS)))]
        dt = DType.from_tag(tag)
        shape = tuple(int(x) for x in rng.integers(0, 5, size=int(rng.integers(0, 3))))
        numel = int(np.prod(shape)) if shape else 1
        name = f"t{i}"
        tensors[name] = fill(rng, dt, numel)
        landing.append([name, off, tag, list(shape)])
        if tag in CONV and rng.random() < 0.5:
            conversions[name] = CONV[tag][int(rng.integers(0, len(CONV[tag])))]
        off += len(tensors[name]) + (int(rng.integers(0, 4)) if rng.random() < 0.3 else 0)
    if rng.random() < 0.05:
        conversions["t0"] = "I32"  # unsupported unless t0 is already I32 -> error or identity
    # every landed range lies inside the buffer; a tight buffer (cap == end of the
    # last landing) overflows when repack padding or a widening cast needs room
    cap = max(1, off + int(rng.integers(0, 64)) if rng.random() > 0.25 else off)
    bounce = int(rng.choice([1, 2, 4, 8, 16, 64], p=[0.04, 0.04, 0.04, 0.28, 0.3, 0.3]))
    return tensors, landing, conversions, cap, bounce


def main():
    rng = np.random.default_rng(0xDE71CE)
    cases = []
    for _ in range(160):
        tensors, landing, conversions, cap, bounce = repack_case(rng)
        pool = DevicePool("host")
        buf = pool.allocate(cap)
        init = rng.integers(0, 256, size=cap, dtype=np.uint8).tobytes()
        buf.write_bytes(0, init)
        for name, off, _tag, _shape in landing:
            if off + len(tensors[name]) <= cap:
                buf.write_bytes(off, tensors[name])
        before = buf.read_bytes(0, cap)
        metas = [(name, off, TensorMetadata(name, DType.from_tag(tag), tuple(shape),
                                            (0, len(tensors[name])))) for name, off, tag, shape in landing]
        case = {"op": "align_and_convert", "input": base64.b64encode(before).decode(), "landing": landing,
                "conversions": conversions, "bounce": bounce}
        try:
            table = align_and_convert(buf, metas, bounce, {k: DType.from_tag(v) for k, v in conversions.items()})
            case["expect"] = {"table": [[n, o, m.dtype.value, list(m.data_offsets)] for n, o, m in table],
                              "sha256": hashlib.sha256(buf.read_bytes(0, cap)).hexdigest()}
        except Exception as e:  # noqa: BLE001 - the class name is the outcome
            case["expect"] = {"error": type(e).__name__}
        cases.append(case)

    for _ in range(80):
        tag = ["F32", "F16", "BF16", "F64", "U8"][int(rng.choice(5, p=[0.3, 0.3, 0.3, 0.05, 0.05]))]
        dt = DType.from_tag(tag)
        target = (CONV.get(tag) or ["F16"])[int(rng.integers(0, len(CONV.get(tag) or ["F16"])))]
        n = int(rng.integers(0, 40))
        begin = int(rng.integers(0, 5)) * (2 if rng.random() < 0.8 else 1)
        raw = fill(rng, dt, n)
        cap = begin + max(len(raw), n * DType.from_tag(target).size_bytes) + int(rng.integers(0, 16))
        if rng.random() < 0.1:
            cap = begin + len(raw)  # widening without room -> OutOfBoundsView
        pool = DevicePool("host")
        buf = pool.allocate(cap)
        buf.write_bytes(0, rng.integers(0, 256, size=cap, dtype=np.uint8).tobytes())
        buf.write_bytes(begin, raw)
        before = buf.read_bytes(0, cap)
        bounce = int(rng.choice([1, 2, 4, 16], p=[0.05, 0.05, 0.1, 0.8]))
        m = TensorMetadata("t", dt, (n,), (begin, begin + len(raw)))
        case = {"op": "convert_dtype", "input": base64.b64encode(before).decode(), "dtype": tag, "numel": n,
                "begin": begin, "target": target, "bounce": bounce}
        try:
            out = convert_dtype(buf, m, DType.from_tag(target), bounce)
            case["expect"] = {"meta": [out.dtype.value, list(out.data_offsets)],
                              "sha256": hashlib.sha256(buf.read_bytes(0, cap)).hexdigest()}
        except Exception as e:  # noqa: BLE001
            case["expect"] = {"error": type(e).__name__}
        cases.append(case)
    (HERE / "device_cases.json").write_text(json.dumps({"cases": cases}) + "\n")
    errs = sum(1 for c in cases if "error" in c["expect"])
    print(f"wrote {len(cases)} cases ({errs} error outcomes)")


if __name__ == "__main__":
    main()
