"""The torch.distributed group (DistGroup) across real processes, on CPU/gloo.

Covers the host-side logic of the N>1 path with world_size 2: control-plane
agreement (the repeated-key probe), the optional ordering check that turns a
cross-rank order mismatch into RendezvousTimeout (ref collective.py:149-159),
in-place broadcast, and the grouped send/recv scatter with uneven remainder
parts reconstructing the source (ref test_collective.py:167-193). On GPUs the
same calls run over NCCL; the shard packing there is the hl_gather kernel,
here the test packs with the oracle's slicing.
"""

from __future__ import annotations

import os
import socket
import sys

import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import numpy as np
    import torch.distributed as dist

    from oracle import oracle
    from paper_2505_23072_b200 import kernels
    from paper_2505_23072_b200.collective import DistGroup, partition
    from paper_2505_23072_b200.errors import RendezvousTimeout
    from paper_2505_23072_b200.format import DType, TensorMetadata

    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        g = DistGroup(check_order=True)
        assert g.world_size == world and g.rank == rank and g.device.type == "cpu"
        # control plane: the owner's verdict reaches everyone
        out["agree"] = g.agree(rank, src=1, value="buffer" if rank == 1 else None, tag="probe:full:k")
        # ordering check: ranks issuing different collectives
        try:
            g.check(("broadcast", "a0" if rank == 0 else "b0", 0))
            out["mismatch"] = "missed"
        except RendezvousTimeout as e:
            out["mismatch"] = "mismatch" in str(e)
        # broadcast in place
        t = torch.arange(10, dtype=torch.uint8) if rank == 0 else torch.zeros(10, dtype=torch.uint8)
        g.broadcast_tensor(t, src=0)
        out["bcast"] = t.tolist()
        # uneven scatter: shape [7, 5] int16 along dim 0 and dim 1 over 2 ranks
        rng = np.random.default_rng(5)
        raw = rng.integers(0, 256, size=7 * 5 * 2, dtype=np.uint8).tobytes()
        for dim in (0, 1):
            m = TensorMetadata("w", DType.I16, (7, 5), (0, len(raw)))
            spec = partition(m, dim, world)
            mine_shape = spec.part_shapes[rank]
            n = int(np.prod(mine_shape)) * 2
            mine = torch.zeros(n, dtype=torch.uint8)
            parts = None
            if rank == 0:
                parts = []
                for r in range(world):
                    _, b = oracle.slice_bytes(raw, "I16", (7, 5), dim, world, r)
                    parts.append(torch.frombuffer(bytearray(b), dtype=torch.uint8))
                mine.copy_(parts[0])
            g.scatter_parts(rank, 0, parts, mine)
            out[f"scatter{dim}"] = (list(mine_shape), bytes(mine.numpy()))
            out["raw"] = raw
        out["bounds"] = [kernels.shard_bounds(7, world, r) for r in range(world)]
        # the bounded (store-counter) barrier the peer-memory plane's close() uses:
        # passes when everyone arrives, raises instead of hanging when a rank never does
        g.bounded_barrier("both", timeout=30)
        out["bounded"] = True
        # a later group over the same ranks meets at fresh keys (its first barrier must
        # still wait for the late rank, not pass on the earlier group's filled counter)
        import time

        g2 = DistGroup(check_order=False)
        if rank == 1:
            time.sleep(1.0)
        t0 = time.monotonic()
        g2.bounded_barrier("both", timeout=30)
        out["second_group_waited"] = rank == 1 or time.monotonic() - t0 > 0.7
        out["alone"] = True
        if rank == 0:
            try:
                g.bounded_barrier("alone", timeout=0.5)
                out["alone"] = "missed"
            except RendezvousTimeout as e:
                out["alone"] = "1 of 2" in str(e)
    finally:
        dist.destroy_process_group()
    q.put((rank, out))


@pytest.mark.timeout(120)
def test_distgroup_two_ranks_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    import numpy as np

    for r in range(world):
        assert res[r]["agree"] == "buffer"
        assert res[r]["mismatch"] is True
        assert res[r]["bcast"] == list(range(10))
        assert res[r]["bounded"] is True and res[r]["alone"] is True
        assert res[r]["second_group_waited"] is True
    raw = res[0]["raw"]
    full = np.frombuffer(raw, dtype=np.int16).reshape(7, 5)
    for dim in (0, 1):
        parts = [np.frombuffer(res[r][f"scatter{dim}"][1], dtype=np.int16).reshape(res[r][f"scatter{dim}"][0])
                 for r in range(world)]
        assert [x.shape[dim] for x in parts] == ([4, 3] if dim == 0 else [3, 2])  # remainder to the lower rank
        assert np.array_equal(np.concatenate(parts, axis=dim), full)
