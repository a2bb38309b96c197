"""Host-side planning and descriptor arithmetic (CPU).

The shard/copy descriptors the loader hands to hl_gather are executed here by
the C oracle (same contract as the kernel) on host memory, and compared with
the reference's slicing; the planner and the realign layout are compared with
the reference's rules and golden tables.
"""

from __future__ import annotations

import numpy as np
import os

import pytest

from conftest import GOLDEN
from oracle import oracle
from paper_2505_23072_b200 import kernels
from paper_2505_23072_b200.collective import partition
from paper_2505_23072_b200.device import DeviceBackend
from paper_2505_23072_b200.errors import BadDim, DimTooSmall, EmptyFileList
from paper_2505_23072_b200.format import DType, TensorMetadata, read_header
from paper_2505_23072_b200.loader import _repack_layout
from paper_2505_23072_b200.transfer import FileSpec, NumaNode, Topology, build_plan, transfer_start, worker_count


def meta(shape, dt=DType.F32):
    n = int(np.prod(shape)) * dt.size_bytes if shape else dt.size_bytes
    return TensorMetadata("t", dt, tuple(shape), (0, n))


def test_partition_reference_rules():
    assert partition(meta((4, 6)), 1, 2).part_shapes == ((4, 3), (4, 3))
    s = partition(meta((4, 7)), 1, 2)
    assert s.part_shapes == ((4, 4), (4, 3)) and s.bounds(0) == (0, 4) and s.bounds(1) == (4, 7)
    with pytest.raises(BadDim):
        partition(meta((4, 6)), 2, 2)
    with pytest.raises(BadDim):
        partition(meta(()), 0, 2)
    with pytest.raises(BadDim):
        partition(meta((4, 6)), -1, 2)
    with pytest.raises(DimTooSmall):
        partition(meta((4, 3)), 1, 4)


def test_shard_bounds_independent_arithmetic(rng):
    for _ in range(200):
        extent = int(rng.integers(1, 100))
        world = int(rng.integers(1, extent + 1))
        assert [kernels.shard_bounds(extent, world, r) for r in range(world)] == oracle.shard_ranges(extent, world)


@pytest.mark.parametrize("dtype", [DType.U8, DType.BF16, DType.F32, DType.I64])
def test_shard_desc_executes_to_reference_slices(rng, dtype):
    lib = oracle.clib()
    if lib is None:
        pytest.skip("oracle not built")
    for _ in range(25):
        nd = int(rng.integers(1, 5))
        shape = tuple(int(rng.integers(1, 7)) for _ in range(nd))
        dim = int(rng.integers(0, nd))
        world = int(rng.integers(1, shape[dim] + 1))
        raw = rng.integers(0, 256, size=int(np.prod(shape)) * dtype.size_bytes, dtype=np.uint8)
        for r in range(world):
            lo, hi = kernels.shard_bounds(shape[dim], world, r)
            exp_shape, exp = oracle.slice_bytes(raw.tobytes(), dtype.value, shape, dim, world, r)
            out = np.zeros(len(exp) + 8, np.uint8)
            d = kernels.shard_desc(raw.ctypes.data, shape, dim, lo, hi, out.ctypes.data, dtype)
            if d[2] and d[3]:
                assert lib.oracle_gather(*d) == 0
            assert out[: len(exp)].tobytes() == exp


def test_algorithmic_bytes():
    d = kernels.copy_desc(0, 0, 100, DType.BF16, DType.F32)
    assert kernels.algorithmic_bytes([d]) == 100 * (2 + 4)


def test_thread_rule_and_plan_tiling():
    topo = Topology((NumaNode(0, physical_cpus=40, device_ids=(0,), storage_ids=(0,)),))
    assert worker_count(9, topo, 0, 16) == 9 and worker_count(72, topo, 0, 16) == 16
    files = [FileSpec("/a", 30_000, 0, 13_281), FileSpec("/b", 5_000, 0, 100)]
    plan = build_plan(files, "simdirect", block_size=1000, topology=topo)
    for spec in plan.buffers:
        blocks = [b for b in plan.blocks if b.buffer_id == spec.buffer_id]
        f = next(x for x in files if x.file_id == spec.file_id)
        start = transfer_start(f.body_offset, DeviceBackend.sim_direct())
        assert start % 512 == 0 and blocks[0].file_off == start
        covered = sorted((b.file_off, b.file_off + b.len) for b in blocks)
        assert covered[0][0] == start and covered[-1][1] == f.size
        assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
        assert all(b.file_off % 512 == 0 for b in blocks)
    host = build_plan(files, "host", block_size=1000, topology=topo)
    assert {b.file_off for b in host.blocks if b.dev_off == 0} == {13_281, 100}
    with pytest.raises(EmptyFileList):
        build_plan([], "host")


def test_loader_repack_layout_matches_reference_tables(golden_cases):
    for case in golden_cases:
        if case["backend"] != "simdirect":
            continue
        for f, offs in case["layouts"].items():
            h = read_header(GOLDEN / "corpora" / f)
            start = h.body_offset // 512 * 512
            landing = {k: h.body_offset + m.begin - start for k, m in h.tensors.items()}
            if all(landing[k] % m.dtype.alignment == 0 for k, m in h.tensors.items()):
                got = landing
            else:
                got, _ = _repack_layout([(k, landing[k], m.dtype, m.nbytes) for k, m in h.tensors.items()])
            assert got == offs, (case["id"], f)


def test_engine_team_shares_node_cores(monkeypatch):
    from paper_2505_23072_b200 import transfer

    monkeypatch.setattr(transfer.os, "sched_getaffinity", lambda pid: set(range(40)))
    monkeypatch.delenv("LOCAL_WORLD_SIZE", raising=False)
    assert transfer.engine_team(16) == 16
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "8")
    assert transfer.engine_team(16) == 4  # floor(0.8 * 40 / 8)
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "64")
    assert transfer.engine_team(16) == transfer.MIN_TEAM  # never fewer than MIN_TEAM readers per rank
    assert transfer.engine_team(2) == 2  # ... unless the cap is lower


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("kind", ["reference", "port"])
def test_bench_cpu_reference_leg(tmp_path, rng, world, kind, monkeypatch):
    """bench.py's reference arm counts exactly the ready bytes of the arm's
    workload (full tensors at W=1, every rank's Megatron-dim slice at W>1),
    through the unmodified reference (aggload from baseline/_ref) or, when
    that is absent, the oracle port; warm and cold passes."""
    import bench
    from paper_2505_23072_b200.format import write_file

    if kind == "port":
        monkeypatch.setattr(bench, "reference_package", lambda: None)
    elif bench.reference_package() is None:
        pytest.skip("baseline/_ref not installed")
    paths, policy, keys, expect = [], {}, [], 0
    for f in range(3):
        tensors = {}
        for i in range(4):
            shape = (6 + i, 10)
            raw = rng.integers(0, 256, int(np.prod(shape)) * 2, dtype=np.uint8).tobytes()
            name = f"f{f}.t{i}"
            tensors[name] = (DType.BF16, shape, raw)
            policy[name] = (None, 0, 1, 0)[i]
            keys.append(name)
            expect += len(raw) * (world if (world > 1 and policy[name] is None) else 1)
        p = tmp_path / f"m{f}.safetensors"
        p.write_bytes(write_file(tensors))
        paths.append(p)
    r = bench.run_cpu_reference(paths, keys, policy, steps=1, warmup=0, cold_steps=1, world=world)
    assert r["kind"] == kind and r["threads"] >= world and r["host_cores"] == os.cpu_count()
    assert f"{expect} ready bytes" in r["sample"]
    assert r["cold"]["residency_before"] == [0.0] or r["cold"]["residency_before"][0] <= 0.01


def test_partition_matches_reference_outcomes():
    """400 random shapes x dims (incl. out of range) x world sizes: same part
    shapes, bounds and rejections as the reference's partition (golden made by
    the reference, tests/golden/partition_cases.json)."""
    import json
    import math

    from paper_2505_23072_b200 import errors

    for c in json.loads((GOLDEN / "partition_cases.json").read_text())["cases"]:
        shape = tuple(c["shape"])
        n = math.prod(shape) if shape else 1
        m = TensorMetadata("k", DType.BF16, shape, (0, 2 * n))
        try:
            spec = partition(m, c["dim"], c["world"])
            got = {"part_shapes": [list(p) for p in spec.part_shapes],
                   "bounds": [list(spec.bounds(r)) for r in range(c["world"])]}
        except errors.AggloadError as e:
            got = {"error": type(e).__name__}
        assert got == c["expect"], c
