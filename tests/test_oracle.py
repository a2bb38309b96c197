"""The CPU oracle pinned against the reference (CPU-only).

* conversions: oracle_c.c and the numpy restatement vs the reference's own
  outputs (tests/golden/conv.npz, from aggload.device._convert_elements);
* known answers quoted from the reference's tests;
* the naive loader and shard slicing vs the reference loader's results on
  the golden corpora (tests/golden/corpora/expect.json);
* the realign relocation table vs the reference's align_fix tables.
"""

from __future__ import annotations

import hashlib
import math
import struct

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle

CORPORA = GOLDEN / "corpora"


@pytest.fixture(scope="module")
def lib():
    lib = oracle.clib()
    if lib is None:
        pytest.skip("oracle/build/liboracle.so not built (make -C oracle)")
    return lib


def _vec(lib, fn, arr):
    f = getattr(lib, fn)
    return np.array([f(int(x)) for x in arr])


def test_c_oracle_exhaustive_16bit(lib, golden_conv):
    all16 = golden_conv["all16"]
    raw = all16.astype("<u2").tobytes()
    assert oracle.convert(raw, "BF16", "F16") == golden_conv["bf16_f16"].tobytes()
    assert oracle.convert(raw, "F16", "F32") == golden_conv["f16_f32"].tobytes()
    assert oracle.convert(raw, "BF16", "F32") == golden_conv["bf16_f32"].tobytes()


def test_c_oracle_f32_sample(lib, golden_conv):
    raw = golden_conv["f32_in"].astype("<u4").tobytes()
    assert oracle.convert(raw, "F32", "F16") == golden_conv["f32_f16"].tobytes()


def test_numpy_restatement_matches_reference_on_non_nan(golden_conv):
    # numpy may take a hardware (F16C / AVX512-FP16) path that quiets NaNs on
    # other CPUs; every non-NaN result must still match the reference bits.
    raw = golden_conv["f32_in"].astype("<u4").tobytes()
    got = np.frombuffer(oracle.convert_numpy(raw, "F32", "F16"), "<u2")
    exp = golden_conv["f32_f16"]
    nan = ((exp & 0x7C00) == 0x7C00) & ((exp & 0x3FF) != 0)
    assert np.array_equal(got[~nan], exp[~nan])
    assert (((got[nan] & 0x7C00) == 0x7C00) & ((got[nan] & 0x3FF) != 0)).all()


@pytest.mark.parametrize("value,half", [(1.0, 0x3C00), (-2.5, 0xC100), (65504.0, 0x7BFF),
                                        (2.0 ** -24, 0x0001), (0.0, 0x0000), (1e30, 0x7C00)])
def test_known_answers_f32_to_f16(lib, value, half):
    # ref pkg/tests/test_device.py:85-90 and :431 (1e30 overflows to inf)
    (bits,) = struct.unpack("<I", struct.pack("<f", value))
    assert lib.oracle_f32_to_f16(bits) == half


@pytest.mark.parametrize("bf16,half", [(0x3F80, 0x3C00), (0x7F80, 0x7C00), (0x7F81, 0x7C08)])
def test_known_answers_bf16_to_f16(lib, bf16, half):
    # ref test_device.py:408-424; 0x7F81 -> 0x7C08 is numpy's NaN payload rule
    assert lib.oracle_f32_to_f16(bf16 << 16) == half


def test_nan_payload_rules(lib):
    assert lib.oracle_f32_to_f16(0x7F800001) == 0x7C01  # payload would vanish: forced non-zero
    assert lib.oracle_f16_to_f32(0x7C01) == 0x7F802000  # widening keeps the payload


def test_oracle_gather_strided_matches_numpy_slicing(lib, rng):
    for _ in range(20):
        shape = tuple(int(rng.integers(1, 9)) for _ in range(3))
        dim = int(rng.integers(0, 3))
        world = int(rng.integers(1, shape[dim] + 1))
        raw = rng.integers(0, 256, size=int(np.prod(shape)) * 4, dtype=np.uint8)
        for r in range(world):
            lo, hi = oracle.shard_ranges(shape[dim], world)[r]
            inner = int(np.prod(shape[dim + 1:]))
            outer = int(np.prod(shape[:dim]))
            out = np.zeros(outer * (hi - lo) * inner * 4, np.uint8)
            if out.size:
                lib.oracle_gather(raw.ctypes.data + lo * inner * 4, out.ctypes.data, outer, (hi - lo) * inner,
                                  shape[dim] * inner * 4, 11, 11)
            assert out.tobytes() == oracle.slice_bytes(raw.tobytes(), "F32", shape, dim, world, r)[1]


def test_naive_oracle_reproduces_reference_loader(golden_cases):
    """oracle.load_all / load_shard_bytes give exactly the bytes the
    reference's loader returned on every rank (hashes in expect.json)."""
    for case in golden_cases:
        files = [CORPORA / f for f in case["files"]]
        owner = {k: f for f in files for k in oracle.read_header(f)[1]}
        full = oracle.load_all(files)
        for rank, got in enumerate(case["ranks"]):
            for key, (kind, shape, digest) in got.items():
                if kind == "full":
                    (_, shp), data = full[key]
                else:
                    shp, data = oracle.load_shard_bytes(owner[key], key, case["dim"], case["world"], rank)
                assert list(shp) == shape and hashlib.sha256(data).hexdigest() == digest, (case["id"], key)


def test_repack_layout_matches_reference_align_fix(golden_cases):
    for case in golden_cases:
        if case["backend"] != "simdirect":
            continue
        for f, offs in case["layouts"].items():
            body, tensors = oracle.read_header(CORPORA / f)
            start = body // 512 * 512
            landing = [(k, body + b - start, dt, e - b) for k, (dt, _, b, e) in tensors.items()]
            aligned = all(off % oracle.SIZES[dt] == 0 for _, off, dt, _ in landing)
            exp = {k: off for k, off, _, _ in landing} if aligned else oracle.repack_layout(landing)
            assert exp == offs, (case["id"], f)


def test_in_place_repack_matches_reference_whole_buffer():
    """The oracle's align_and_convert restatement reproduces the reference's
    whole buffer (sha256) and table on every successful device_cases.json case
    (tests/golden/make_device_golden.py ran the reference itself)."""
    import base64
    import json

    from conftest import GOLDEN

    n = 0
    for c in json.loads((GOLDEN / "device_cases.json").read_text())["cases"]:
        if c["op"] != "align_and_convert" or "error" in c["expect"]:
            continue
        landing = [(k, off, dt, math.prod(shape)) for k, off, dt, shape in c["landing"]]
        table, out = oracle.align_and_convert_bytes(base64.b64decode(c["input"]), landing, c["conversions"])
        assert [[k, o, dt] for k, o, dt in table] == [t[:3] for t in c["expect"]["table"]], c
        assert hashlib.sha256(out).hexdigest() == c["expect"]["sha256"], c
        n += 1
    assert n > 100


def test_cpu_loader_port_round_trip(tmp_path, rng):
    from conftest import random_tensor_set
    from paper_2505_23072_b200.format import write_file

    t = random_tensor_set(rng, 8, prefix="c")
    p = tmp_path / "c.safetensors"
    p.write_bytes(write_file(t))
    ld = oracle.CpuLoader([p], block=4096, bounce=1000)
    ld.copy()
    for k, (dt, shape, raw) in t.items():
        assert ld.get_tensor(k).tobytes() == raw
    assert oracle.thread_rule(9, cpus=40) == 9 and oracle.thread_rule(72, cpus=40) == 16
