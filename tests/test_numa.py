"""NUMA placement rule of the engine without a GPU (hl_topology_resolve,
ref transfer.py:51-121 Topology and 274-293 worker affinity): the node is the
caller's request, else $HL_NUMA_NODE, else the GPU's PCI numa_node; the
workers and the pinned ring are bound to that node's CPUs the process may
use. A fake two-node sysfs tree under $HL_SYSFS_ROOT stands in for a
dual-socket 8-GPU host."""

from __future__ import annotations

import os

import pytest

from paper_2505_23072_b200 import _native

BUS = "0000:1B:00.0"


@pytest.fixture
def fake_sysfs(tmp_path, monkeypatch):
    dev = tmp_path / "sys/bus/pci/devices" / BUS.lower()
    dev.mkdir(parents=True)
    (dev / "numa_node").write_text("1\n")
    allowed = sorted(os.sched_getaffinity(0))
    half = max(1, len(allowed) // 2)
    nodes = {0: allowed[:half], 1: allowed[half:] or allowed[:1]}
    for node, cpus in nodes.items():
        d = tmp_path / f"sys/devices/system/node/node{node}"
        d.mkdir(parents=True)
        d.joinpath("cpulist").write_text(",".join(map(str, cpus)) + ",4095\n")  # 4095: not ours
    monkeypatch.setenv("HL_SYSFS_ROOT", str(tmp_path))
    monkeypatch.delenv("HL_NUMA_NODE", raising=False)
    return nodes


def test_gpu_node_from_pci_sysfs(fake_sysfs):
    node, cpus = _native.topology_resolve(BUS)
    assert node == 1 and cpus == fake_sysfs[1]  # disallowed CPUs dropped


def test_env_override_beats_pci_node(fake_sysfs, monkeypatch):
    monkeypatch.setenv("HL_NUMA_NODE", "0")
    assert _native.topology_resolve(BUS) == (0, fake_sysfs[0])


def test_explicit_request_beats_env(fake_sysfs, monkeypatch):
    monkeypatch.setenv("HL_NUMA_NODE", "0")
    assert _native.topology_resolve(BUS, requested_node=1) == (1, fake_sysfs[1])


def test_unknown_device_or_node_means_unpinned(fake_sysfs):
    assert _native.topology_resolve("0000:ff:00.0") == (-1, [])
    assert _native.topology_resolve(BUS, requested_node=7) == (7, [])


def test_engine_team_keeps_four_readers_per_rank(monkeypatch):
    from paper_2505_23072_b200 import transfer

    monkeypatch.setenv("LOCAL_WORLD_SIZE", "8")
    assert transfer.engine_team() >= min(transfer.MIN_TEAM, transfer.DEFAULT_WORKER_CAP)
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "1")
    assert transfer.engine_team() >= transfer.engine_team.__defaults__[0] * 0 + 1


def test_storage_node_from_the_block_device(tmp_path, monkeypatch):
    """hl_storage_numa_node: the file's st_dev -> /sys/dev/block/MAJ:MIN ->
    the nearest device-tree ancestor with a numa_node (the NVMe PCI function)."""
    path = tmp_path / "f.bin"
    path.write_bytes(b"x")
    st = os.stat(path)
    root = tmp_path / "fake"
    pci = root / "sys/devices/pci0000:80/0000:80:01.0"
    blk = pci / "nvme/nvme1/nvme1n1"
    blk.mkdir(parents=True)
    (pci / "numa_node").write_text("1\n")
    links = root / "sys/dev/block"
    links.mkdir(parents=True)
    (links / f"{os.major(st.st_dev)}:{os.minor(st.st_dev)}").symlink_to(
        "../../devices/pci0000:80/0000:80:01.0/nvme/nvme1/nvme1n1")
    monkeypatch.setenv("HL_SYSFS_ROOT", str(root))
    assert _native.storage_numa_node(str(path)) == 1
    (pci / "numa_node").write_text("-1\n")
    assert _native.storage_numa_node(str(path)) == -1
    assert _native.storage_numa_node(str(tmp_path / "missing")) == -1
    monkeypatch.setenv("HL_SYSFS_ROOT", str(tmp_path / "nowhere"))
    assert _native.storage_numa_node(str(path)) == -1
