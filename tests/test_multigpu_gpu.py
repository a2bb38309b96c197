"""Cross-device paths, run whenever the box has more than one GPU (skipped on
the 1-GPU boxes): thread ranks on cuda:0..N-1 (every rank's kernel reads its
owner's HBM in place over NVLink: hl_enable_peer_access), and one process per
GPU over NCCL on both data planes — ncclBroadcast / grouped send-recv and
CUDA-IPC peer pulls — all against the reference loader's own outputs
(tests/golden/corpora/expect.json, ref collective.py:175-255)."""

from __future__ import annotations

import hashlib
import json
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

from conftest import GOLDEN, ROOT, run_ranks  # noqa: E402

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs at least 2 GPUs")]

CORPORA = GOLDEN / "corpora"


def _cases(world):
    return [c for c in json.loads((CORPORA / "expect.json").read_text())["cases"] if c["world"] == world]


def _retrieve(fb, world, dim):
    got = {}
    for k in sorted(fb.keys()):
        m = fb.metadata(k)
        if world > 1 and dim < len(m.shape) and m.shape[dim] >= world:
            v, kind = fb.get_sharded(k, dim), "shard"
        else:
            v, kind = fb.get_tensor(k), "full"
        got[k] = [kind, list(v.shape), hashlib.sha256(v.tobytes()).hexdigest(), v.torch.device.index]
    return got


@pytest.mark.parametrize("world", [2, 3, 4])
def test_thread_ranks_on_distinct_gpus(world):
    from paper_2505_23072_b200 import LoaderConfig, ProcessGroup, SafeTensorsFileLoader

    n = torch.cuda.device_count()
    for case in _cases(world):
        mapping = {int(r): [str(CORPORA / f) for f in fs] for r, fs in case["mapping"].items()}
        group = ProcessGroup(world)

        def rank_main(rank):
            loader = SafeTensorsFileLoader(group, f"cuda:{rank % n}", rank=rank,
                                           config=LoaderConfig(backend=case["backend"]))
            loader.add_filenames(mapping)
            got = _retrieve(loader.copy_files_to_device(), world, case["dim"])
            loader.close()
            return got

        for rank, got in enumerate(run_ranks(world, rank_main)):
            assert all(v[3] == rank % n for v in got.values())
            assert {k: v[:3] for k, v in got.items()} == case["ranks"][rank], (case["id"], rank)


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2505_23072_b200 import DistGroup, LoaderConfig, SafeTensorsFileLoader

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    out = {}
    try:
        for plane in ("nccl", "ipc"):
            group = DistGroup(device=torch.device("cuda", rank), data_plane=plane, check_order=True)
            for case in _cases(world):
                mapping = {int(r): [str(CORPORA / f) for f in fs] for r, fs in case["mapping"].items()}
                loader = SafeTensorsFileLoader(group, config=LoaderConfig(backend=case["backend"]))
                loader.add_filenames(mapping)
                got = _retrieve(loader.copy_files_to_device(), world, case["dim"])
                loader.close()
                out[(plane, case["id"])] = ({k: v[:3] for k, v in got.items()} == case["ranks"][rank]
                                            and all(v[3] == rank for v in got.values()))
    except BaseException as e:  # noqa: BLE001
        import traceback

        out = ("error", f"{type(e).__name__}: {e}\n{traceback.format_exc()}")
    finally:
        dist.destroy_process_group()
    q.put((rank, out))


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world", [2, 4])
def test_nccl_and_ipc_planes_one_process_per_gpu(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    port = _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=800) for _ in range(world))
    for p in procs:
        p.join(60)
    for r in range(world):
        assert not (isinstance(res[r], tuple) and res[r][0] == "error"), res[r]
        assert res[r] and all(res[r].values()), res[r]
