"""Shared fixtures. `-m gpu` tests need a B200 (they call through the C ABI);
everything else runs on CPU: the oracle against the reference's golden
vectors, host planning logic, the ABI's symbol table, and gloo multi-process
tests of the torch.distributed group."""

from __future__ import annotations

import json
import sys
import threading
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhbmload.so")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture
def rng():
    return np.random.default_rng(0xB200)


@pytest.fixture(scope="session")
def golden_cases():
    return json.loads((GOLDEN / "corpora" / "expect.json").read_text())["cases"]


@pytest.fixture(scope="session")
def golden_conv():
    return dict(np.load(GOLDEN / "conv.npz"))


# ---------------------------------------------------------------- corpus helpers
DIMS = [0, 1, 1, 2, 2, 3, 3, 4, 5, 7, 8, 13, 16, 64]


def random_tensor_set(rng, n, prefix="t", dtypes=None, max_rank=4, max_numel=65536):
    """name -> (DType, shape, raw bytes); every dtype, rank 0-4, skewed dims."""
    from paper_2505_23072_b200.format import DType

    dtypes = dtypes or list(DType)
    out = {}
    for i in range(n):
        dt = dtypes[int(rng.integers(0, len(dtypes)))]
        rank = int(rng.integers(0, max_rank + 1))
        shape = tuple(int(rng.choice(DIMS)) for _ in range(rank))
        while max_numel is not None and int(np.prod(shape, dtype=np.int64)) > max_numel:
            shape = tuple(min(d, 4) for d in shape)
        nb = int(np.prod(shape, dtype=np.int64)) * dt.size_bytes if shape else dt.size_bytes
        out[f"{prefix}{i}"] = (dt, shape, rng.integers(0, 256, size=nb, dtype=np.uint8).tobytes())
    return out


def pad_for_body_residue(tensors, residue):
    """pad_header_to so that body_offset % 512 == residue."""
    layout = {k: {"dtype": dt.value, "shape": list(s), "data_offsets": [0, 0]} for k, (dt, s, _) in tensors.items()}
    natural = len(json.dumps(layout, separators=(",", ":")).encode())
    base = natural + 128
    return base + (residue - (8 + base) % 512) % 512


class RankFailure(Exception):
    def __init__(self, rank, exc):
        super().__init__(f"rank {rank} raised {type(exc).__name__}: {exc}")
        self.rank = rank
        self.exc = exc


def run_ranks(world, fn, join_timeout=120.0):
    """fn(rank) on `world` threads (thread ranks of one ProcessGroup)."""
    from paper_2505_23072_b200.errors import RendezvousTimeout

    results, failures = [None] * world, {}

    def runner(r):
        try:
            results[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            failures[r] = e

    ts = [threading.Thread(target=runner, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(join_timeout)
    if any(t.is_alive() for t in ts):
        raise TimeoutError("rank threads still running")
    if failures:
        primary = [r for r, e in failures.items() if not isinstance(e, RendezvousTimeout)]
        r = min(primary) if primary else min(failures)
        raise RankFailure(r, failures[r]) from failures[r]
    return results
