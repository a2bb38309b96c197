"""The multi-GPU data planes across real processes (DistGroup).

ipc: the peer-memory plane (the default on one node).

W processes share the box's one B200 (CUDA IPC works between processes on the
same device; the control plane is gloo on 127.0.0.1). Every rank lands only
its own files, publishes the buffer once, and then every get_tensor /
get_sharded is ONE hl_gather launch per rank reading the owner's HBM through
the IPC mapping — on a multi-GPU box the same reads travel over NVLink.
Results are checked against the reference loader's own outputs
(tests/golden/corpora/expect.json) and the oracle.

nccl: the collective plane (owner pack kernel + broadcast / grouped
send-recv). NCCL refuses two ranks on one GPU, so gloo stands in for it here:
the same calls, gloo moving the CUDA tensors (P2P staged through the host).
"""

from __future__ import annotations

import hashlib
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

from conftest import GOLDEN, ROOT  # noqa: E402

pytestmark = pytest.mark.gpu

CORPORA = GOLDEN / "corpora"


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, job, q):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, job(rank, world)))
    except BaseException as e:  # noqa: BLE001
        import traceback

        q.put((rank, ("error", f"{type(e).__name__}: {e}\n{traceback.format_exc()}")))
    finally:
        dist.destroy_process_group()


def _run(world, job, timeout=240):
    port = _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, job, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, v = q.get(timeout=timeout)
        res[r] = v
    for p in procs:
        p.join(60)
    for r, v in res.items():
        if isinstance(v, tuple) and v and v[0] == "error":
            raise AssertionError(f"rank {r}: {v[1]}")
    return [res[r] for r in range(world)]


def golden_job(rank, world, plane="ipc", batched=False):
    """Every golden case of this world size through the given data plane,
    key by key or as one get_tensors batch per case."""
    import json

    from paper_2505_23072_b200 import DistGroup, LoaderConfig, SafeTensorsFileLoader

    cases = [c for c in json.loads((CORPORA / "expect.json").read_text())["cases"] if c["world"] == world]
    group = DistGroup(device=torch.device("cuda", 0), data_plane=plane, check_order=True)
    out = {}
    for case in cases:
        mapping = {int(r): [str(CORPORA / f) for f in fs] for r, fs in case["mapping"].items()}
        for auto in (True, False):
            loader = SafeTensorsFileLoader(group, config=LoaderConfig(backend=case["backend"], auto_release=auto))
            loader.add_filenames(mapping)
            fb = loader.copy_files_to_device()
            got = {}
            keys = sorted(fb.keys())
            dims = {k: case["dim"] for k in keys
                    if case["dim"] < len(fb.metadata(k).shape) and fb.metadata(k).shape[case["dim"]] >= world}
            views = fb.get_tensors(keys, dims=dims) if batched else {
                k: (fb.get_sharded(k, dims[k]) if k in dims else fb.get_tensor(k)) for k in keys}
            for k in keys:
                v = views[k]
                got[k] = ["shard" if k in dims else "full", list(v.shape), hashlib.sha256(v.tobytes()).hexdigest()]
            fb.close()
            loader.close()
            out[(case["id"], auto)] = got == case["ranks"][rank]
    return out


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.timeout(600)
def test_ipc_plane_matches_reference_loader(world):
    for rank_result in _run(world, golden_job):
        assert rank_result and all(rank_result.values()), rank_result


def golden_job_collective_plane(rank, world):
    return golden_job(rank, world, plane="nccl")


def golden_job_collective_plane_batched(rank, world):
    return golden_job(rank, world, plane="nccl", batched=True)


def golden_job_ipc_batched(rank, world):
    return golden_job(rank, world, plane="ipc", batched=True)


def golden_job_ipc_peer_tma(rank, world):
    """Peer pulls through the TMA kernels (HL_PEER_TMA): key by key and batched."""
    from paper_2505_23072_b200 import kernels

    kernels.PEER_TMA = True
    out = golden_job(rank, world, plane="ipc")
    out.update({(k, "batched"): v for k, v in golden_job(rank, world, plane="ipc", batched=True).items()})
    return out


def golden_job_collective_plane_batched_bcast(rank, world):
    from paper_2505_23072_b200 import loader

    loader.BIG_BROADCAST = 0  # every replicated tensor through the broadcast branch
    return golden_job(rank, world, plane="nccl", batched=True)


@pytest.mark.parametrize("job", ["collective", "collective_bcast", "ipc", "ipc_peer_tma"])
@pytest.mark.timeout(600)
def test_batched_planes_match_reference_loader(job):
    """get_tensors as ONE batch per case: the collective plane's single
    owner-side launch + grouped point-to-point call, and the ipc plane's
    single pull launch, against the reference loader's outputs."""
    fn = {"collective": golden_job_collective_plane_batched, "ipc": golden_job_ipc_batched,
          "ipc_peer_tma": golden_job_ipc_peer_tma,
          "collective_bcast": golden_job_collective_plane_batched_bcast}[job]
    for rank_result in _run(3, fn):
        assert rank_result and all(rank_result.values()), rank_result


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.timeout(600)
def test_collective_plane_matches_reference_loader(world):
    """The NCCL data plane's whole flow (owner pack kernel, broadcast, grouped
    send/recv, repeated/stale keys) with gloo standing in for NCCL — NCCL
    refuses two ranks on one GPU, and the box has one."""
    for rank_result in _run(world, golden_job_collective_plane):
        assert rank_result and all(rank_result.values()), rank_result


def features_job(rank, world, plane="ipc"):
    """dtype casts, Megatron dims on a larger checkpoint slice, repeated keys
    (buffer still alive, then from a surviving tensor), stale shards."""
    import numpy as np

    from oracle import oracle
    from paper_2505_23072_b200 import DistGroup, SafeTensorsFileLoader
    from paper_2505_23072_b200.errors import StaleKey
    from paper_2505_23072_b200.format import DType, write_file

    d = f"/tmp/hl_ipc_feat_{os.getppid()}"
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(77)
    files = []
    for i in range(world):
        t = {f"l{i}.q": (DType.BF16, (256, 192), rng.integers(0, 256, 256 * 192 * 2, dtype=np.uint8).tobytes()),
             f"l{i}.o": (DType.F32, (96, 130), rng.integers(0, 256, 96 * 130 * 4, dtype=np.uint8).tobytes()),
             f"l{i}.n": (DType.BF16, (192,), rng.integers(0, 256, 384, dtype=np.uint8).tobytes())}
        p = f"{d}/f{i}.safetensors"
        if rank == 0:
            with open(p, "wb") as f:
                f.write(write_file(t, pad_header_to=301 + i))  # odd bodies: realign on simdirect
        files.append((p, t))
    torch.distributed.barrier()
    group = DistGroup(device=torch.device("cuda", 0), data_plane=plane)
    loader = SafeTensorsFileLoader(group, "simdirect")
    loader.add_filenames({r: [files[r][0]] for r in range(world)})
    fb = loader.copy_files_to_device()
    ok = {}
    keep = []
    for i, (p, t) in enumerate(files):
        q = fb.get_sharded(f"l{i}.q", 0, dtype=torch.float16)
        conv = oracle.convert(t[f"l{i}.q"][2], "BF16", "F16")
        ok[f"q{i}"] = q.tobytes() == oracle.slice_bytes(conv, "F16", (256, 192), 0, world, rank)[1]
        o = fb.get_sharded(f"l{i}.o", 1)
        ok[f"o{i}"] = o.tobytes() == oracle.slice_bytes(t[f"l{i}.o"][2], "F32", (96, 130), 1, world, rank)[1]
        n1 = fb.get_tensor(f"l{i}.n")
        n2 = fb.get_tensor(f"l{i}.n")  # repeated: served again
        ok[f"n{i}"] = n1.tobytes() == n2.tobytes() == t[f"l{i}.n"][2]
        keep.append(n1)
        try:
            fb.get_sharded(f"l{i}.o", 1)  # buffer released after its last key: stale
            ok[f"stale{i}"] = False
        except StaleKey:
            ok[f"stale{i}"] = True
    fb.close()
    loader.close()

    # batched: one pull launch per rank for a whole "layer" of keys
    from paper_2505_23072_b200 import _native

    loader = SafeTensorsFileLoader(group, "host")
    loader.add_filenames({r: [files[r][0]] for r in range(world)})
    fb = loader.copy_files_to_device()
    keys = [f"l{i}.{x}" for i in range(world) for x in ("q", "o", "n")]
    dims = {k: (0 if k.endswith("q") else 1) for k in keys if not k.endswith("n")}
    l0 = _native.kernel_launches()
    got = fb.get_tensors(keys, dims=dims)
    if plane == "ipc":  # the collective plane serves a batch key by key
        ok["batch_launches"] = _native.kernel_launches() - l0 <= 3  # one per conversion kind present
    for i, (p, t) in enumerate(files):
        ok[f"bq{i}"] = got[f"l{i}.q"].tobytes() == oracle.slice_bytes(t[f"l{i}.q"][2], "BF16", (256, 192), 0, world, rank)[1]
        ok[f"bo{i}"] = got[f"l{i}.o"].tobytes() == oracle.slice_bytes(t[f"l{i}.o"][2], "F32", (96, 130), 1, world, rank)[1]
        ok[f"bn{i}"] = got[f"l{i}.n"].tobytes() == t[f"l{i}.n"][2]
    fb.close()
    loader.close()
    return ok


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.timeout(600)
def test_ipc_plane_casts_dims_repeats(world):
    for rank_result in _run(world, features_job):
        assert all(rank_result.values()), rank_result


def features_job_collective_plane(rank, world):
    return features_job(rank, world, plane="nccl")


@pytest.mark.timeout(600)
def test_collective_plane_casts_dims_repeats():
    for rank_result in _run(3, features_job_collective_plane):
        assert all(rank_result.values()), rank_result


def auto_plane_job(rank, world):
    """data_plane="auto" probes CUDA IPC once (every rank maps its neighbour's
    probe allocation and reads it with hl_gather) and settles on "ipc" here."""
    from paper_2505_23072_b200 import DistGroup

    g = DistGroup(device=torch.device("cuda", 0))
    return {"plane": g.data_plane}


@pytest.mark.parametrize("world", [2, 4])
def test_auto_plane_probes_ipc(world):
    assert [r["plane"] for r in _run(world, auto_plane_job)] == ["ipc"] * world


def vllm_iter_job(rank, world):
    """vllm_loader.weights_iterator under torch.distributed (vLLM's TP
    workers): files spread over the ranks, every rank gets every tensor."""
    import numpy as np

    from paper_2505_23072_b200.format import DType, write_file
    from paper_2505_23072_b200.vllm_loader import weights_iterator

    d = f"/tmp/hl_vllm_iter_{os.getppid()}"
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(5)
    tensors, files = {}, []
    for i in range(3):
        t = {f"m{i}.w": (DType.BF16, (64, 48), rng.integers(0, 256, 64 * 48 * 2, dtype=np.uint8).tobytes()),
             f"m{i}.b": (DType.F32, (48,), rng.integers(0, 256, 48 * 4, dtype=np.uint8).tobytes())}
        tensors.update(t)
        p = f"{d}/model-{i + 1:05d}-of-00003.safetensors"
        if rank == 0:
            with open(p, "wb") as f:
                f.write(write_file(t))
        files.append(p)
    torch.distributed.barrier()
    got = {}
    for name, t in weights_iterator(files):
        got[name] = t.contiguous().view(torch.uint8).cpu().numpy().tobytes() == tensors[name][2]
    return {"all_keys": set(got) == set(tensors), **got}


def test_vllm_iterator_multirank():
    for rank_result in _run(2, vllm_iter_job):
        assert all(rank_result.values()), rank_result


def ops_job(rank, world, plane, batched=False):
    """Replay every reference op trace of this world size (tests/golden/ops_cases.json)
    through DistGroup on the given data plane; outcomes must equal the reference's.
    batched: runs of fresh keys go through one get_tensors call."""
    import json

    from paper_2505_23072_b200 import DistGroup, LoaderConfig, SafeTensorsFileLoader
    from paper_2505_23072_b200.transfer import NumaNode, Topology
    from test_ops_gpu import runs_of, step

    group = DistGroup(device=torch.device("cuda", 0), data_plane=plane)
    result = {}
    for ci, case in enumerate(json.loads((GOLDEN / "ops_cases.json").read_text())["cases"]):
        if case["world"] != world:
            continue
        files = [GOLDEN / "corpora" / f for f in case["files"]]
        mapping = {r: [str(p) for i, p in enumerate(files) if i % world == r] for r in range(world)}
        topo = Topology((NumaNode(0, 32, tuple(range(world)), (0,)),))
        ld = SafeTensorsFileLoader(group, config=LoaderConfig(backend=case["backend"], topology=topo,
                                                              auto_release=case["auto_release"]))
        ld.add_filenames(mapping)
        fb = ld.copy_files_to_device()
        held, trace = {}, []
        runs = runs_of(case, 0) if batched else {}
        i = 0
        while i < len(case["ops"]):
            i = step(fb, case["ops"], i, held, trace, runs)
        fb.close()
        ld.close()
        exp = case["ranks"][rank]
        bad = [(j, case["ops"][j], g, e) for j, (g, e) in enumerate(zip(trace, exp)) if g != e]
        result[ci] = True if not bad else str(bad[0])
    return result


def ops_job_ipc(rank, world):
    return ops_job(rank, world, "ipc")


def ops_job_collective(rank, world):
    return ops_job(rank, world, "nccl")


def ops_job_ipc_batched(rank, world):
    return ops_job(rank, world, "ipc", batched=True)


def ops_job_collective_batched(rank, world):
    return ops_job(rank, world, "nccl", batched=True)


@pytest.mark.parametrize("plane", ["ipc", "collective", "ipc_batched", "collective_batched"])
@pytest.mark.timeout(900)
def test_planes_replay_reference_op_traces(plane):
    fn = {"ipc": ops_job_ipc, "collective": ops_job_collective, "ipc_batched": ops_job_ipc_batched,
          "collective_batched": ops_job_collective_batched}[plane]
    for world in (2, 3, 4):
        for rank_result in _run(world, fn, timeout=600):
            bad = {k: v for k, v in rank_result.items() if v is not True}
            assert rank_result and not bad, (world, bad)


def fanout_job(rank, world):
    """The peer-memory plane's broadcast route (loader._fanout_route): at
    W >= 3 replicated tensors over BIG_BROADCAST go through the broadcast
    instead of W-1 peer pulls. BIG_BROADCAST = 0 sends every replicated
    tensor that way: golden corpora key by key and batched, and every
    reference op trace (repeated / stale / survivor keys)."""
    from paper_2505_23072_b200 import loader

    loader.BIG_BROADCAST = 0
    out = {("keys",) + k: v for k, v in golden_job(rank, world, plane="ipc").items()}
    out.update({("batch",) + k: v for k, v in golden_job(rank, world, plane="ipc", batched=True).items()})
    out.update({("ops", k): v for k, v in ops_job(rank, world, "ipc").items()})
    out.update({("ops_batched", k): v for k, v in ops_job(rank, world, "ipc", batched=True).items()})
    return out


@pytest.mark.parametrize("world", [3, 4])
@pytest.mark.timeout(900)
def test_ipc_plane_fanout_route_matches_reference(world):
    for rank_result in _run(world, fanout_job, timeout=800):
        bad = {k: v for k, v in rank_result.items() if v is not True}
        assert rank_result and not bad, (world, bad)
