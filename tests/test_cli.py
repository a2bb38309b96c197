"""The CLI (paper_2505_23072_b200.cli), mirroring the reference's test_cli.py:
gen / inspect / shard-plan on CPU (byte- and document-identical to the
reference's own outputs, tests/golden/cli_gen.json), bench on the GPU."""

from __future__ import annotations

import hashlib
import json
import math
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT
from paper_2505_23072_b200.cli import main
from paper_2505_23072_b200.format import DType, read_header, validate, write_file


def run_cli(capsys, *argv):
    rc = main([str(a) for a in argv])
    cap = capsys.readouterr()
    return rc, cap.out, cap.err


# ------------------------------------------------------------------------------ golden
CASES = json.loads((GOLDEN / "cli_gen.json").read_text())["cases"]


@pytest.mark.parametrize("case", CASES, ids=[" ".join(c["args"]) for c in CASES])
def test_gen_inspect_plan_match_reference(tmp_path, capsys, case):
    rc, *_ = run_cli(capsys, "gen", *case["args"], "--out", tmp_path)
    assert rc == 0
    files = sorted(tmp_path.glob("*.safetensors"))
    assert [f.name for f in files] == case["files"]
    assert [hashlib.sha256(f.read_bytes()).hexdigest() for f in files] == case["sha256"]
    rc, out, _ = run_cli(capsys, "inspect", files[0])
    assert rc == 0 and json.loads(out) == case["inspect"]
    for tag, want in case["shard_plan"].items():
        w, d = tag[1:].split("d")
        rc, out, _ = run_cli(capsys, "shard-plan", files[0], "--world-size", w, "--dim", d)
        got = json.loads(out)
        assert rc == 0 and got.pop("file") == str(files[0]) and got == want


# ---------------------------------------------------------------------- reference tests
def test_gen_files_parse_and_validate(tmp_path, capsys):
    rc, *_ = run_cli(capsys, "gen", "--files", 2, "--bytes-per-file", 65536, "--seed", 7, "--out", tmp_path / "c")
    assert rc == 0
    files = sorted((tmp_path / "c").glob("*.safetensors"))
    assert len(files) == 2
    for f in files:
        h = read_header(f)
        validate(h, h.file_size)
        assert h.file_size - h.body_offset == 65536 and h.body_offset % 512 == 0


def test_gen_deterministic(tmp_path, capsys):
    digests = []
    for sub in ("one", "two"):
        assert run_cli(capsys, "gen", "--files", 2, "--bytes-per-file", 4096, "--seed", 42, "--dtype", "mixed",
                       "--out", tmp_path / sub)[0] == 0
        digests.append([hashlib.sha256(f.read_bytes()).hexdigest()
                        for f in sorted((tmp_path / sub).glob("*.safetensors"))])
    assert digests[0] == digests[1]


def test_gen_pad_header_and_suffix(tmp_path, capsys):
    assert run_cli(capsys, "gen", "--files", 2, "--bytes-per-file", 1024, "--pad-header", 299,
                   "--out", tmp_path / "odd")[0] == 0
    assert all(read_header(f).body_offset == 307 for f in (tmp_path / "odd").glob("*.safetensors"))
    assert run_cli(capsys, "gen", "--files", 1, "--bytes-per-file", "64k", "--out", tmp_path / "k")[0] == 0
    h = read_header(next((tmp_path / "k").glob("*.safetensors")))
    assert h.file_size - h.body_offset == 65536


def test_inspect_errors(tmp_path, capsys):
    bad = tmp_path / "bad.safetensors"
    bad.write_bytes(b"\xff\x00\x00\x00\x00\x00\x00\x00{}")  # declares 255 header bytes, has 2
    rc, _, err = run_cli(capsys, "inspect", bad)
    assert rc == 1 and "TruncatedHeader" in err
    rc, _, _ = run_cli(capsys, "inspect", tmp_path / "nope.safetensors")
    assert rc == 2


def test_shard_plan_remainder_and_bad_dim(tmp_path, capsys):
    p = tmp_path / "plan.safetensors"
    shapes = {"even": (4, 6), "odd": (4, 7), "s": (), "ok": (8, 2)}
    p.write_bytes(write_file({k: (DType.F32, s, bytes(4 * math.prod(s))) for k, s in shapes.items()}))
    rc, out, _ = run_cli(capsys, "shard-plan", p, "--world-size", 2, "--dim", 1)
    doc = json.loads(out)
    assert rc == 0
    assert doc["keys"]["even"]["part_shapes"] == [[4, 3], [4, 3]]
    assert doc["keys"]["odd"]["part_shapes"] == [[4, 4], [4, 3]]
    assert doc["keys"]["s"]["error"] == "BadDim"
    rc, out, _ = run_cli(capsys, "shard-plan", p, "--world-size", 2, "--dim", 0)
    assert json.loads(out)["keys"]["ok"]["part_shapes"] == [[4, 2], [4, 2]]


def test_bench_missing_corpus(tmp_path, capsys):
    rc, _, err = run_cli(capsys, "bench", "--dir", tmp_path / "empty")
    assert rc == 2 and "EmptyFileList" in err


def test_module_entrypoint(tmp_path):
    out = subprocess.run([sys.executable, "-m", "paper_2505_23072_b200", "gen", "--files", "1", "--bytes-per-file",
                          "1024", "--out", str(tmp_path)], capture_output=True, text=True, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    p = subprocess.run([sys.executable, "-m", "paper_2505_23072_b200", "inspect",
                        str(next(tmp_path.glob("*.safetensors")))], capture_output=True, text=True, cwd=ROOT)
    assert p.returncode == 0 and json.loads(p.stdout)["tensors"]


def test_expected_bytes_slicing(tmp_path):
    """The bench's verifier slices like the reference's load_shard_bytes
    (reference.py:56-66): remainder rows/cols to lower ranks, row-major."""
    import numpy as np

    from paper_2505_23072_b200.cli import expected_bytes

    a = np.arange(2 * 5 * 3, dtype=np.int16).reshape(2, 5, 3)
    p = tmp_path / "x.safetensors"
    p.write_bytes(write_file({"a": (DType.I16, a.shape, a.tobytes())}))
    meta = read_header(p).tensors["a"]
    assert expected_bytes(str(p), meta, None, 2, 0) == a.tobytes()
    assert expected_bytes(str(p), meta, 1, 2, 0) == np.ascontiguousarray(a[:, 0:3]).tobytes()
    assert expected_bytes(str(p), meta, 1, 2, 1) == np.ascontiguousarray(a[:, 3:5]).tobytes()
    assert expected_bytes(str(p), meta, 2, 2, 1) == np.ascontiguousarray(a[:, :, 2:3]).tobytes()


# --------------------------------------------------------------------------------- GPU
@pytest.fixture
def corpus(tmp_path, capsys):
    d = tmp_path / "corpus"
    run_cli(capsys, "gen", "--files", 4, "--bytes-per-file", 65536, "--seed", 3, "--dtype", "mixed", "--out", d)
    return d


@pytest.mark.gpu
def test_bench_world_one(corpus, capsys):
    rc, out, err = run_cli(capsys, "bench", "--dir", corpus, "--backend", "host", "--workers", 2, "--repeat", 2)
    assert rc == 0, err
    doc = json.loads(out)
    assert set(doc) == {"elapsed_seconds", "bytes", "throughput_bytes_per_sec", "workers", "block_size", "backend",
                        "world_size", "per_rank", "cross_numa_blocks"}
    assert doc["world_size"] == 1 and doc["backend"] == "host"
    assert doc["bytes"] == 4 * 65536  # host transfers exactly the bodies
    assert doc["throughput_bytes_per_sec"] == pytest.approx(doc["bytes"] / doc["elapsed_seconds"], rel=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("backend", ["host", "simdirect", "gds"])
def test_bench_two_ranks_verified(corpus, capsys, backend):
    rc, out, err = run_cli(capsys, "bench", "--dir", corpus, "--world-size", 2, "--dim", 1, "--repeat", 1,
                           "--backend", backend, "--auto-release")
    assert rc == 0, err  # rc 4 = a rank's bytes differ from the file
    doc = json.loads(out)
    assert doc["backend"] == backend and len(doc["per_rank"]) == 2
    assert sum(e["files"] for e in doc["per_rank"]) == 4
    for e in doc["per_rank"]:
        assert abs(e["bytes"] - doc["bytes"] / 2) <= 65536 + 8 + 4096


@pytest.mark.gpu
def test_bench_topology_env(corpus, tmp_path, capsys, monkeypatch):
    topo = tmp_path / "topo.json"
    topo.write_text(json.dumps({"nodes": [{"node_id": 0, "physical_cpus": 1, "device_ids": [0], "storage_ids": [0]}]}))
    monkeypatch.setenv("AGGLOAD_TOPOLOGY", str(topo))
    rc, out, err = run_cli(capsys, "bench", "--dir", corpus, "--workers", 8, "--repeat", 1)
    assert rc == 0, err
    assert json.loads(out)["workers"] == 1  # a 1-CPU node caps the reference worker rule at one thread
