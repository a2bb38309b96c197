"""The in-process rank group's control plane on CPU (ref tests/test_collective.py):
rendezvous, ordering-bug detection, timeouts and poisoning, agree, and the
argument checks of broadcast/scatter that fire before any data moves. The data
moves themselves (GPU kernels) are covered in test_loader_gpu / test_acceptance_gpu."""

from __future__ import annotations

import random
import threading
import time

import pytest

from paper_2505_23072_b200.collective import ProcessGroup, SingleGroup, partition
from paper_2505_23072_b200.errors import RendezvousTimeout, SpecMismatch
from paper_2505_23072_b200.format import DType, TensorMetadata


def run_ranks(world, fn, timeout=20.0):
    """fn(rank) on one thread per rank; returns {rank: result or exception}."""
    out = {}

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            out[r] = e

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert all(not t.is_alive() for t in ts), "a rank hung"
    return out


def meta(shape):
    n = 1
    for d in shape:
        n *= d
    return TensorMetadata("k", DType.F32, tuple(shape), (0, 4 * n))


def test_exchange_everyone_sees_everything():
    g = ProcessGroup(4)
    res = run_ranks(4, lambda r: g.exchange(r, r * 10))
    assert all(res[r] == {0: 0, 1: 10, 2: 20, 3: 30} for r in range(4))


def test_world_one_identity():
    g = SingleGroup()
    assert g.exchange(0, "x") == {0: "x"}
    assert g.agree(0, 0, 5) == 5
    token = object()
    assert g.broadcast(0, token, src=0) is token
    assert g.scatter(0, partition(meta((4, 2)), 0, 1), 0, token) is token


def test_rank_out_of_range():
    g = ProcessGroup(2)
    with pytest.raises(ValueError):
        g.exchange(2, None)
    with pytest.raises(ValueError):
        ProcessGroup(0)


def test_agree_distributes_src_value():
    g = ProcessGroup(3)
    res = run_ranks(3, lambda r: g.agree(r, src=1, value=f"from{r}", tag="t"))
    assert res == {0: "from1", 1: "from1", 2: "from1"}


def test_missing_rank_times_out_and_poisons():
    g = ProcessGroup(2, timeout=0.3)
    t0 = time.monotonic()
    with pytest.raises(RendezvousTimeout, match="timed out"):
        g.exchange(0, "alone")
    assert time.monotonic() - t0 < 5
    with pytest.raises(RendezvousTimeout):  # poisoned: later collectives fail fast
        g.exchange(1, "late")


def test_order_mismatch_detected_on_every_rank():
    g = ProcessGroup(2)
    res = run_ranks(2, lambda r: g.agree(r, src=0, value=1, tag=("a" if r == 0 else "b")))
    assert all(isinstance(res[r], RendezvousTimeout) for r in range(2))
    assert "ordering bug" in str(res[0])


def test_abort_releases_waiters():
    g = ProcessGroup(3, timeout=30)

    def fn(r):
        if r == 2:
            time.sleep(0.2)
            g.abort("rank 2 failed: boom")
            return "aborted"
        return g.exchange(r, r)

    res = run_ranks(3, fn, timeout=10)
    assert res[2] == "aborted"
    assert all(isinstance(res[r], RendezvousTimeout) and "boom" in str(res[r]) for r in (0, 1))


def test_out_of_turn_collective_poisons():
    g = ProcessGroup(2, timeout=5)
    box = {}

    def first():
        try:
            g.exchange(0, "a")
        except RendezvousTimeout as e:
            box["waiter"] = e

    t = threading.Thread(target=first, daemon=True)
    t.start()
    time.sleep(0.1)
    with pytest.raises(RendezvousTimeout, match="out of turn"):
        g.exchange(0, "again")
    t.join(5)
    assert isinstance(box.get("waiter"), RendezvousTimeout)


def test_randomized_delays_never_deadlock():
    world, rounds = 4, 40
    g = ProcessGroup(world, timeout=20)
    rng = [random.Random(r) for r in range(world)]

    def fn(r):
        seen = []
        for i in range(rounds):
            time.sleep(rng[r].random() * 0.002)
            got = g.exchange(r, (i, r))
            assert got == {q: (i, q) for q in range(world)}
            seen.append(g.agree(r, src=i % world, value=i * 100 + r, tag=str(i)))
        return seen

    res = run_ranks(world, fn, timeout=60)
    for r in range(world):
        assert res[r] == [i * 100 + i % world for i in range(rounds)]


def test_scatter_world_mismatch_before_any_data_move():
    g = ProcessGroup(2)
    spec = partition(meta((4, 2)), 0, 3)
    with pytest.raises(SpecMismatch):
        g.scatter(0, spec, 0, None)


def test_broadcast_bad_src():
    g = ProcessGroup(2)
    with pytest.raises(ValueError):
        g.broadcast(0, None, src=2)
