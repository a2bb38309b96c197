"""API-semantics parity: random op sequences (get_tensor / get_sharded on
live, repeated, dropped and stale keys, unknown keys, bad dims, close, reads
after close) replayed on the B200 loader must give exactly the outcomes the
REFERENCE loader gave — same bytes (sha256) and shapes, or the same error
class — on every rank (tests/golden/ops_cases.json, made by the reference:
tests/golden/make_ops_golden.py). Thread ranks share the one GPU."""

from __future__ import annotations

import gc
import hashlib
import json
import threading

import pytest

torch = pytest.importorskip("torch")

from conftest import GOLDEN  # noqa: E402
from paper_2505_23072_b200 import LoaderConfig, ProcessGroup, SafeTensorsFileLoader  # noqa: E402
from paper_2505_23072_b200.transfer import NumaNode, Topology  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = json.loads((GOLDEN / "ops_cases.json").read_text())["cases"]


def runs_of(case, rank):
    """Maximal runs of consecutive get_tensor/get_sharded ops on distinct,
    never-requested keys that the reference served without error: each run
    can be ONE get_tensors batch (same results and consumption as the ops)."""
    ops, exp = case["ops"], case["ranks"][rank]
    seen, runs, i = set(), {}, 0
    while i < len(ops):
        j, keys = i, set()
        while (j < len(ops) and ops[j][0] in ("tensor", "shard") and exp[j][0] == "ok"
               and ops[j][1] not in seen and ops[j][1] not in keys):
            keys.add(ops[j][1])
            j += 1
        if j - i >= 2:
            runs[i] = j
        for k in range(i, max(j, i + 1)):
            if ops[k][0] in ("tensor", "shard"):
                seen.add(ops[k][1])
        i = max(j, i + 1)
    return runs


def step(fb, ops, i, held, trace, runs):
    """Execute op i (or the batch starting at i); returns the next op index."""
    op = ops[i]
    if i in runs:
        j = runs[i]
        keys = [ops[k][1] for k in range(i, j)]
        dims = {ops[k][1]: ops[k][2] for k in range(i, j) if ops[k][0] == "shard"}
        got = fb.get_tensors(keys, dims=dims)
        for k in range(i, j):
            v = got[ops[k][1]]
            held[k] = v
            trace.append(["ok", list(v.shape), hashlib.sha256(v.tobytes()).hexdigest()])
        return j
    try:
        if op[0] in ("tensor", "shard"):
            v = fb.get_tensor(op[1]) if op[0] == "tensor" else fb.get_sharded(op[1], op[2])
            held[i] = v
            trace.append(["ok", list(v.shape), hashlib.sha256(v.tobytes()).hexdigest()])
        elif op[0] == "drop":
            held.pop(op[1], None)
            gc.collect()
            trace.append(["ok"])
        elif op[0] == "read":
            v = held.get(op[1])
            trace.append(["ok", hashlib.sha256(v.tobytes()).hexdigest()] if v is not None else ["ok"])
        elif op[0] == "close":
            fb.close()
            trace.append(["ok"])
    except Exception as e:  # noqa: BLE001 - the class name is the outcome
        trace.append(["err", type(e).__name__])
    return i + 1


def replay(case, batched=False, backend=None):
    files = [GOLDEN / "corpora" / f for f in case["files"]]
    world = case["world"]
    mapping = {r: [str(p) for i, p in enumerate(files) if i % world == r] for r in range(world)}
    topo = Topology((NumaNode(0, 32, tuple(range(world)), (0,)),))
    group = ProcessGroup(world, timeout=60)
    out, errors = [None] * world, {}

    def rank_main(rank):
        try:
            ld = SafeTensorsFileLoader(group, rank=rank, config=LoaderConfig(
                backend=backend or case["backend"], topology=topo, auto_release=case["auto_release"]))
            ld.add_filenames(mapping)
            fb = ld.copy_files_to_device()
            held, trace = {}, []
            runs = runs_of(case, 0) if batched else {}  # the same grouping on every rank
            i = 0
            while i < len(case["ops"]):
                i = step(fb, case["ops"], i, held, trace, runs)
            out[rank] = trace
            fb.close()
            ld.close()
        except BaseException:  # noqa: BLE001
            import traceback

            errors[rank] = traceback.format_exc()

    ts = [threading.Thread(target=rank_main, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
    assert not errors, errors
    return out


@pytest.mark.parametrize("batched", [False, True])
@pytest.mark.parametrize("i", range(len(CASES)))
def test_op_sequence_matches_reference(i, batched):
    """batched: runs of fresh keys go through ONE get_tensors call instead."""
    case = CASES[i]
    got = replay(case, batched)
    for rank in range(case["world"]):
        for j, (g, e) in enumerate(zip(got[rank], case["ranks"][rank])):
            assert g == e, (f"rank {rank} op {j} {case['ops'][j]}: got {g}, reference {e}", case["backend"],
                            case["auto_release"], case["world"])


SIMDIRECT = [i for i, c in enumerate(CASES) if c["backend"] == "simdirect"]


@pytest.mark.parametrize("i", SIMDIRECT)
def test_gds_landing_matches_reference_simdirect_traces(i):
    """The GDS-shaped landing (4 KiB floors instead of the reference's 512) is
    invisible to the API: the reference's simdirect traces replay unchanged."""
    case = CASES[i]
    got = replay(case, batched=bool(i % 2), backend="gds")
    for rank in range(case["world"]):
        assert got[rank] == case["ranks"][rank], (rank, i)
