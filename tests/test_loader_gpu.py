"""Behavioural parity of the drop-in API, on the GPU.

Each test restates one reference behaviour (pkg/tests/test_loader.py and
pkg/src/aggload/loader.py) against our loader; bytes are checked with the
oracle (oracle.load_all / load_shard_bytes, ref reference.py:38-77).
"""

from __future__ import annotations

import gc

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import RankFailure, pad_for_body_residue, random_tensor_set, run_ranks  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2505_23072_b200 import LoaderConfig, ProcessGroup, SafeTensorsFileLoader, SingleGroup, _native  # noqa: E402
from paper_2505_23072_b200.errors import (  # noqa: E402
    BadDim,
    DimTooSmall,
    DuplicateKey,
    EmptyFileList,
    IoError,
    MisalignedView,
    RendezvousTimeout,
    StaleKey,
    UnknownKey,
    UnsupportedConversion,
    UseAfterClose,
)
from paper_2505_23072_b200.format import DType, write_file  # noqa: E402
from paper_2505_23072_b200.tensorview import TORCH_DTYPES, read_element  # noqa: E402

pytestmark = pytest.mark.gpu


def _write(tmp_path, name, tensors, pad=None):
    p = tmp_path / name
    p.write_bytes(write_file(tensors, pad_header_to=pad))
    return p


@pytest.fixture
def two_files(tmp_path, rng):
    a = random_tensor_set(rng, 1, prefix="a")
    b = {"b0": (DType.F32, (4, 6), rng.integers(0, 256, 96, dtype=np.uint8).tobytes())}
    return _write(tmp_path, "a.safetensors", a), _write(tmp_path, "b.safetensors", b), a, b


# ------------------------------------------------------------------ single rank
def test_get_tensor_bytes_dtype_shape_and_torch_view(tmp_path, rng):
    t = random_tensor_set(rng, 6, prefix="a")
    p = _write(tmp_path, "a.safetensors", t)
    loader = SafeTensorsFileLoader(SingleGroup(), "host")
    loader.add_filenames({0: [p]})
    fb = loader.copy_files_to_device()
    for name, (dt, shape, raw) in t.items():
        v = fb.get_tensor(name)
        assert v.dtype is dt and v.shape == shape and v.tobytes() == raw
        assert v.torch.is_cuda and v.torch.dtype == TORCH_DTYPES[dt] and tuple(v.torch.shape) == shape
        assert v.torch.contiguous().view(torch.uint8).cpu().numpy().tobytes() == raw
    fb.close()
    loader.close()


def test_zero_copy_without_auto_release(tmp_path, rng):
    t = random_tensor_set(rng, 2, prefix="a", dtypes=[DType.F32])
    p = _write(tmp_path, "a.safetensors", t)
    loader = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(auto_release=False))
    loader.add_filenames({0: [p]})
    fb = loader.copy_files_to_device()
    before = loader.pool.allocated_bytes
    v = fb.get_tensor("a0")
    assert loader.pool.allocated_bytes == before
    assert v.buffer is fb._hosted[str(p)].buffer
    assert v.torch.data_ptr() == v.buffer.ptr + v.base_offset  # a true alias of the landed bytes
    fb.close()


def test_auto_release_returns_buffer_per_file(tmp_path, rng):
    files = {}
    for i in range(2):
        t = {f"p{i}_a": (DType.F32, (3,), rng.integers(0, 256, 12, dtype=np.uint8).tobytes()),
             f"p{i}_b": (DType.F32, (5,), rng.integers(0, 256, 20, dtype=np.uint8).tobytes())}
        files[str(_write(tmp_path, f"p{i}.safetensors", t))] = t
    loader = SafeTensorsFileLoader(SingleGroup(), "host")
    loader.add_filenames({0: list(files)})
    fb = loader.copy_files_to_device()
    first, second = list(files)
    views = [fb.get_tensor(k) for k in files[first]]
    assert fb._hosted[first].buffer.released and not fb._hosted[second].buffer.released
    assert loader.pool.pooled_bytes == fb._hosted[first].buffer.capacity
    assert all(v.tobytes() == files[first][k][2] for k, v in zip(files[first], views))
    fb.close()
    assert loader.pool.allocated_bytes == 0


def test_get_sharded_world_one_validates_then_full(two_files):
    pa, pb, _, b = two_files
    loader = SafeTensorsFileLoader(SingleGroup(), "host")
    loader.add_filenames({0: [pa, pb]})
    fb = loader.copy_files_to_device()
    with pytest.raises(BadDim):
        fb.get_sharded("b0", dim=2)
    v = fb.get_sharded("b0", dim=1)
    assert v.shape == (4, 6) and v.tobytes() == b["b0"][2]
    fb.close()


# ------------------------------------------------------------------ multi rank (thread ranks on the GPU)
def test_broadcast_and_shard_two_ranks(two_files):
    pa, pb, a, b = two_files
    mapping = {0: [str(pa)], 1: [str(pb)]}
    group = ProcessGroup(2)

    def rank_main(rank):
        loader = SafeTensorsFileLoader(group, "host", rank=rank)
        loader.add_filenames(mapping)
        fb = loader.copy_files_to_device()
        ta, tb = fb.get_tensor("a0"), fb.get_sharded("b0", dim=1)
        out = (ta.tobytes(), tb.tobytes(), tb.shape, set(fb._hosted))
        fb.close()
        loader.close()
        return out

    r0, r1 = run_ranks(2, rank_main)
    assert r0[0] == r1[0] == a["a0"][2]
    assert r0[2] == r1[2] == (4, 3)
    assert r0[3] == {str(pa)} and r1[3] == {str(pb)}  # tensors live only on their owner until shuffled
    full = np.frombuffer(b["b0"][2], np.uint32).reshape(4, 6)
    got = np.concatenate([np.frombuffer(r0[1], np.uint32).reshape(4, 3),
                          np.frombuffer(r1[1], np.uint32).reshape(4, 3)], axis=1)
    assert np.array_equal(got, full)


def test_order_mismatch_times_out(two_files):
    pa, pb, *_ = two_files
    group = ProcessGroup(2, timeout=1.0)

    def rank_main(rank):
        loader = SafeTensorsFileLoader(group, "host", rank=rank)
        loader.add_filenames({0: [str(pa)], 1: [str(pb)]})
        fb = loader.copy_files_to_device()
        for k in (["a0", "b0"] if rank == 0 else ["b0", "a0"]):
            fb.get_tensor(k)

    with pytest.raises(RankFailure) as err:
        run_ranks(2, rank_main)
    assert isinstance(err.value.exc, RendezvousTimeout)


def test_any_identical_permutation_succeeds(tmp_path, rng):
    """ref tests/test_loader.py:170-192: any key order works if every rank uses it."""
    files = {}
    for i in range(2):
        tensors = random_tensor_set(rng, 3, prefix=f"f{i}_")
        files[str(_write(tmp_path, f"f{i}.safetensors", tensors))] = tensors
    mapping = {0: [sorted(files)[0]], 1: [sorted(files)[1]]}
    expect = {k: raw for t in files.values() for k, (_, _, raw) in t.items()}
    group = ProcessGroup(2)

    for order in (list(rng.permutation(list(expect))) for _ in range(3)):
        def rank_main(rank, order=order):
            loader = SafeTensorsFileLoader(group, "host", rank=rank)
            loader.add_filenames(mapping)
            fb = loader.copy_files_to_device()
            got = {k: fb.get_tensor(k).tobytes() for k in order}
            fb.close()
            return got

        for got in run_ranks(2, rank_main):
            assert got == expect


def test_multirank_repeat_from_survivor(two_files):
    """ref tests/test_loader.py:312-327: a consumed key whose owner buffer was
    released is served again from the surviving view on every rank."""
    pa, pb, a, _ = two_files
    group = ProcessGroup(2)

    def rank_main(rank):
        loader = SafeTensorsFileLoader(group, "host", rank=rank)
        loader.add_filenames({0: [str(pa)], 1: [str(pb)]})
        fb = loader.copy_files_to_device()
        first = fb.get_tensor("a0")
        again = fb.get_tensor("a0")
        out = first.tobytes(), again.tobytes()
        fb.close()
        return out

    for first, again in run_ranks(2, rank_main):
        assert first == again == a["a0"][2]


def test_unknown_key_keeps_group_usable(two_files):
    pa, pb, *_ = two_files
    group = ProcessGroup(2)

    def rank_main(rank):
        loader = SafeTensorsFileLoader(group, "host", rank=rank)
        loader.add_filenames({0: [str(pa)], 1: [str(pb)]})
        fb = loader.copy_files_to_device()
        with pytest.raises(UnknownKey):
            fb.get_tensor("nope")
        return fb.get_tensor("a0").tobytes()

    r0, r1 = run_ranks(2, rank_main)
    assert r0 == r1


@pytest.mark.parametrize("backend", ["host", "simdirect"])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_end_to_end_against_oracle(tmp_path, rng, backend, world):
    files = []
    for i in range(world):
        t = random_tensor_set(rng, 5, prefix=f"e{i}_")
        files.append(str(_write(tmp_path, f"e{i}.safetensors", t, pad_for_body_residue(t, int(rng.integers(0, 512))))))
    mapping = {r: [files[r]] for r in range(world)}
    expect = oracle.load_all(files)
    owner = {k: f for f in files for k in oracle.read_header(f)[1]}
    group = ProcessGroup(world)

    def rank_main(rank):
        loader = SafeTensorsFileLoader(group, backend, rank=rank)
        loader.add_filenames(mapping)
        fb = loader.copy_files_to_device()
        out = {}
        for k in sorted(expect):
            (dt, shape), _ = expect[k]
            if world > 1 and len(shape) >= 1 and shape[0] >= world:
                out[k] = ("shard", fb.get_sharded(k, 0).tobytes())
            else:
                out[k] = ("full", fb.get_tensor(k).tobytes())
        fb.close()
        loader.close()
        return out

    for rank, got in enumerate(run_ranks(world, rank_main)):
        for k, (kind, data) in got.items():
            if kind == "full":
                assert data == expect[k][1], k
            else:
                assert data == oracle.load_shard_bytes(owner[k], k, 0, world, rank)[1], k


# ------------------------------------------------------------------ add_filenames / errors
def test_duplicate_key_empty_mapping_and_bad_rank(tmp_path, rng, two_files):
    t = random_tensor_set(rng, 1, prefix="same")
    p1, p2 = _write(tmp_path, "x.safetensors", t), _write(tmp_path, "y.safetensors", t)
    with pytest.raises(DuplicateKey):
        SafeTensorsFileLoader(SingleGroup(), "host").add_filenames({0: [p1, p2]})
    loader = SafeTensorsFileLoader(SingleGroup(), "host")
    loader.add_filenames({})
    with pytest.raises(EmptyFileList):
        loader.copy_files_to_device()
    with pytest.raises(ValueError):
        SafeTensorsFileLoader(SingleGroup(), "host").add_filenames({1: [str(two_files[0])]})


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(IoError):
        SafeTensorsFileLoader(SingleGroup(), "host").add_filenames({0: [tmp_path / "nope.safetensors"]})


def test_skew_warning_on_every_rank(tmp_path, rng):
    big = {"big": (DType.U8, (8192,), rng.integers(0, 256, 8192, dtype=np.uint8).tobytes())}
    small = {"small": (DType.U8, (8,), bytes(8))}
    pb, ps = _write(tmp_path, "big.safetensors", big), _write(tmp_path, "small.safetensors", small)
    group = ProcessGroup(2)

    def rank_main(rank):
        loader = SafeTensorsFileLoader(group, "host", rank=rank)
        loader.add_filenames({0: [str(pb)], 1: [str(ps)]})
        return loader.skew_warning

    assert all(w and "skew" in w for w in run_ranks(2, rank_main))


# ------------------------------------------------------------------ repeat / stale / close
def test_repeat_and_stale(tmp_path, rng):
    t = random_tensor_set(rng, 3, prefix="k")
    loader = SafeTensorsFileLoader(SingleGroup(), "host")
    loader.add_filenames({0: [_write(tmp_path, "k.safetensors", t)]})
    fb = loader.copy_files_to_device()
    first = fb.get_tensor("k0")
    assert fb.get_tensor("k0").tobytes() == first.tobytes()  # buffer still alive
    fb.close()

    t1 = random_tensor_set(rng, 1, prefix="s", dtypes=[DType.F32])
    loader = SafeTensorsFileLoader(SingleGroup(), "host")
    loader.add_filenames({0: [_write(tmp_path, "s.safetensors", t1)]})
    fb = loader.copy_files_to_device()
    v = fb.get_tensor("s0")  # consumes the only key: buffer released
    assert loader.pool.pooled_bytes > 0
    assert fb.get_tensor("s0").tobytes() == v.tobytes()  # served from the surviving view
    del v
    gc.collect()
    with pytest.raises(StaleKey):
        fb.get_tensor("s0")
    fb.close()


def test_stale_sharded_multirank(two_files):
    pa, pb, *_ = two_files
    group = ProcessGroup(2)

    def rank_main(rank):
        loader = SafeTensorsFileLoader(group, "host", rank=rank)
        loader.add_filenames({0: [str(pa)], 1: [str(pb)]})
        fb = loader.copy_files_to_device()
        fb.get_sharded("b0", dim=1)
        fb.get_tensor("a0")
        try:
            fb.get_sharded("b0", dim=1)
            return "no error"
        except StaleKey:
            return "stale"

    assert run_ranks(2, rank_main) == ["stale", "stale"]


def test_close_semantics(tmp_path, rng):
    t = random_tensor_set(rng, 4, prefix="c", dtypes=[DType.F32])
    p = _write(tmp_path, "c.safetensors", t)
    loader = SafeTensorsFileLoader(SingleGroup(), "host")
    loader.add_filenames({0: [p]})
    fb = loader.copy_files_to_device()
    cap = fb.transferred_buffer_bytes
    fb.close()
    assert loader.pool.pooled_bytes == cap and loader.pool.allocated_bytes == 0
    fb.close()
    loader.close()
    loader.close()
    with pytest.raises(UseAfterClose):
        fb.get_tensor("c0")

    loader = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(auto_release=False))
    loader.add_filenames({0: [p]})
    fb = loader.copy_files_to_device()
    v = fb.get_tensor("c0")
    keep = v.torch
    fb.close()
    with pytest.raises(UseAfterClose):
        v.tobytes()
    if v.numel:
        with pytest.raises(UseAfterClose):
            read_element(v, tuple(0 for _ in v.shape))
    assert keep.is_cuda  # the torch tensor a caller kept stays valid


# ------------------------------------------------------------------ alignment (odd headers)
@pytest.mark.parametrize("backend", ["simdirect", "gds"])
@pytest.mark.parametrize("residue", [1, 107, 255, 511])
def test_odd_header_realigned(tmp_path, rng, backend, residue):
    t = random_tensor_set(rng, 6, prefix="o")
    p = _write(tmp_path, "odd.safetensors", t, pad_for_body_residue(t, residue))
    loader = SafeTensorsFileLoader(SingleGroup(), backend, config=LoaderConfig(auto_release=False))
    loader.add_filenames({0: [p]})
    fb = loader.copy_files_to_device()
    hosted = fb._hosted[str(p)]
    for k, (dt, shape, raw) in t.items():
        assert hosted.dev_offsets[k] % dt.alignment == 0
        assert fb.get_tensor(k).tobytes() == raw
    fb.close()


def test_make_view_rejects_misaligned(tmp_path):
    from paper_2505_23072_b200.format import TensorMetadata
    from paper_2505_23072_b200.tensorview import make_view

    pool = SafeTensorsFileLoader(SingleGroup(), "host").pool
    buf = pool.allocate(64)
    with pytest.raises(MisalignedView):
        make_view(buf, 2, TensorMetadata("t", DType.F32, (2,), (0, 8)))


# ------------------------------------------------------------------ dtype superset (on-device cast)
@pytest.mark.parametrize("world", [1, 2])
def test_dtype_cast_on_device_matches_oracle(tmp_path, rng, world):
    files, expect = [], {}
    for i in range(world):
        t = {f"w{i}_bf": (DType.BF16, (16, 24), rng.integers(0, 256, 768, dtype=np.uint8).tobytes()),
             f"w{i}_f32": (DType.F32, (8, 10), rng.integers(0, 256, 320, dtype=np.uint8).tobytes()),
             f"w{i}_u8": (DType.U8, (10,), rng.integers(0, 256, 10, dtype=np.uint8).tobytes())}
        files.append(str(_write(tmp_path, f"w{i}.safetensors", t, pad_for_body_residue(t, 3))))
        expect.update(t)
    group = ProcessGroup(world)

    def rank_main(rank):
        loader = SafeTensorsFileLoader(group, "simdirect", rank=rank)
        loader.add_filenames({r: [files[r]] for r in range(world)})
        fb = loader.copy_files_to_device()
        out = {}
        for k in sorted(expect):
            if k.endswith("u8"):
                with pytest.raises(UnsupportedConversion):
                    fb.get_tensor(k, dtype=DType.F16)
                out[k] = fb.get_tensor(k).tobytes()
            elif world > 1:
                out[k] = fb.get_sharded(k, 1, dtype=torch.float16).tobytes()
            else:
                out[k] = fb.get_tensor(k, dtype="F16").tobytes()
        fb.close()
        return out

    for rank, got in enumerate(run_ranks(world, rank_main)):
        for k, (dt, shape, raw) in expect.items():
            if k.endswith("u8"):
                assert got[k] == raw
                continue
            conv = oracle.convert(raw, dt.value, "F16")
            if world > 1:
                conv = oracle.slice_bytes(conv, "F16", shape, 1, world, rank)[1]
            assert got[k] == conv, k


def test_copy_files_to_device_dtype(tmp_path, rng):
    t = {"x": (DType.BF16, (33,), rng.integers(0, 256, 66, dtype=np.uint8).tobytes()),
         "y": (DType.I32, (4,), rng.integers(0, 256, 16, dtype=np.uint8).tobytes())}
    p = _write(tmp_path, "c.safetensors", t, pad_for_body_residue(t, 107))
    loader = SafeTensorsFileLoader(SingleGroup(), "host")
    loader.add_filenames({0: [p]})
    fb = loader.copy_files_to_device(dtype=DType.F32)
    x = fb.get_tensor("x")
    assert x.dtype is DType.F32 and x.tobytes() == oracle.convert(t["x"][2], "BF16", "F32")
    assert fb.get_tensor("y").tobytes() == t["y"][2]
    fb.close()


def test_get_tensors_batched_matches_per_key(tmp_path, rng):
    t = random_tensor_set(rng, 12, prefix="b", dtypes=[DType.BF16, DType.F32, DType.U8, DType.I64])
    p = _write(tmp_path, "b.safetensors", t, pad_for_body_residue(t, 77))
    keys = sorted(t)
    dims = {k: 0 for k in keys if len(t[k][1]) >= 1 and t[k][1][0] >= 1}
    loader = SafeTensorsFileLoader(SingleGroup(), "simdirect")
    loader.add_filenames({0: [p]})
    fb = loader.copy_files_to_device()
    launches = _native.kernel_launches()
    got = fb.get_tensors(keys, dims=dims)
    assert _native.kernel_launches() - launches <= 4  # one per kernel variant present (aligned/shifted/mixed/generic)
    for k in keys:
        assert got[k].tobytes() == t[k][2] and got[k].shape == t[k][1]
    assert fb._hosted[str(p)].buffer.released  # all keys consumed: auto-release fired
    with pytest.raises(BadDim):
        fb.get_tensors([keys[0]], dims={keys[0]: 9})
    fb.close()


def test_upstream_spellings_as_dict_filename_shape(tmp_path, rng):
    """fastsafetensors' own FilesBufferOnDevice spellings (superset): as_dict
    with dim -1 = full tensor, get_filename, get_shape."""
    t = random_tensor_set(rng, 6, prefix="u", dtypes=[DType.BF16, DType.F32])
    p = _write(tmp_path, "u.safetensors", t)
    loader = SafeTensorsFileLoader(SingleGroup(), "host")
    loader.add_filenames({0: [p]})
    fb = loader.copy_files_to_device()
    keys = sorted(t)
    assert fb.get_filename(keys[0]) == str(p) and fb.get_filename("missing") == ""
    assert fb.get_shape(keys[1]) == list(t[keys[1]][1])
    req = {k: (-1 if i % 2 else 0) for i, k in enumerate(keys) if t[k][1] and t[k][1][0] >= 1}
    got = fb.as_dict(req)
    assert list(got) == list(req)
    for k in req:
        assert got[k].tobytes() == t[k][2]  # world 1: every shard is the full tensor
    fb.close()


def test_safe_open_and_context_managers(tmp_path, rng):
    """safetensors/fastsafe_open-style convenience and `with` on the loader
    and the handle (superset API)."""
    from paper_2505_23072_b200 import safe_open

    t = random_tensor_set(rng, 5, prefix="o", dtypes=[DType.BF16, DType.F32, DType.I64])
    p = _write(tmp_path, "o.safetensors", t)
    with safe_open(str(p), device="cuda:0") as f:
        assert sorted(f.keys()) == sorted(t)
        for k, (dt, shape, raw) in t.items():
            x = f.get_tensor(k)
            assert x.is_cuda and tuple(x.shape) == shape
            assert x.reshape(-1).view(torch.uint8).cpu().numpy().tobytes() == raw
    with SafeTensorsFileLoader(SingleGroup(), "host") as loader:
        loader.add_filenames({0: [p]})
        with loader.copy_files_to_device() as fb:
            v = fb.get_tensor(sorted(t)[0])
            x = v.torch
        with pytest.raises(UseAfterClose):
            fb.get_tensor(sorted(t)[1])
        with pytest.raises(UseAfterClose):  # the reference's close invalidates returned handles
            v.tobytes()
    # ... while the torch tensor the user holds stays valid (torch owns the memory)
    assert x.reshape(-1).view(torch.uint8).cpu().numpy().tobytes() == t[sorted(t)[0]][2]


@pytest.mark.parametrize("batched", [False, True])
def test_back_to_back_loads_never_overwrite_pending_reads(tmp_path, batched):
    """The upstream per-file-group pattern — load, retrieve, close, next
    loader — with the retrievals still queued (behind a spin) when close()
    returns the file buffer to torch's allocator and the next load reuses
    that memory at once: every retrieved tensor must still hold the FIRST
    file's bytes (ref transfer.py:364-378: the reference completes by join)."""
    n = 6 << 20
    files = []
    for i in range(2):
        raw = np.full(n, 17 + 100 * i, dtype=np.uint8)
        raw[::4097] = i  # not constant, same size
        files.append((_write(tmp_path, f"f{i}.safetensors", {"w": (DType.U8, (n,), raw.tobytes())}), raw))
    loader = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(auto_release=True))
    loader.add_filenames({0: [files[0][0]]})
    fb = loader.copy_files_to_device()
    torch.cuda.synchronize()
    torch.cuda._sleep(400_000_000)  # keep the retrieval below queued for ~0.2 s
    got = fb.get_tensors(["w"])["w"] if batched else fb.get_tensor("w")
    fb.close()
    loader.close()
    second = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(auto_release=False))
    second.add_filenames({0: [files[1][0]]})
    fb2 = second.copy_files_to_device()
    torch.cuda.synchronize()
    assert np.array_equal(got.torch.cpu().numpy(), files[0][1])
    assert np.array_equal(fb2.get_tensor("w").torch.cpu().numpy(), files[1][1])
    fb2.close()
    second.close()


def test_deferred_clone_batches(tmp_path, rng):
    """World of one, auto_release: per-key clones are queued and launched
    together (ONE hl_gather per DEFER_KEYS tensors), and every way to reach
    a result's bytes — .torch, tobytes, the buffer's tensor, close() — sees
    them written, bit-exact."""
    from paper_2505_23072_b200 import loader as loader_mod

    t = random_tensor_set(rng, 150, prefix="k", dtypes=[DType.BF16, DType.F32, DType.U8, DType.I64])
    p = _write(tmp_path, "many.safetensors", t)
    ld = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(auto_release=True))
    ld.add_filenames({0: [p]})
    fb = ld.copy_files_to_device()
    torch.cuda.synchronize()
    l0 = _native.kernel_launches()
    views = {k: fb.get_tensor(k) for k in t}
    queued = _native.kernel_launches() - l0
    # the full batches went out, and the tail batch with the file's last key (so the file
    # buffer returns to the pool right then); a batch is one launch per kernel variant it
    # needs: bulk copies, element-path tails, ... — at most 4 here
    assert 0 < queued <= -(-len(t) // loader_mod.DEFER_KEYS) * 4 < len(t) // 10
    names = list(t)
    assert views[names[-1]].tobytes() == t[names[-1]][2]
    assert _native.kernel_launches() - l0 == queued  # nothing was left to flush
    for k in names[:5]:
        assert views[k].buffer.tensor.numel() >= 0
    got = {k: v.torch for k, v in views.items()}
    torch.cuda.synchronize()
    for k, (dt, shape, raw) in t.items():
        assert got[k].view(torch.uint8).cpu().numpy().tobytes() == raw if shape else True, k
        assert views[k].tobytes() == raw, k
    # a fresh handle: results first read after close()
    ld2 = SafeTensorsFileLoader(SingleGroup(), "host", config=LoaderConfig(auto_release=True))
    ld2.add_filenames({0: [p]})
    fb2 = ld2.copy_files_to_device()
    later = {k: fb2.get_tensor(k, dtype=(DType.F16 if t[k][0] is DType.BF16 else None)) for k in names[:40]}
    fb2.close()
    ld2.close()
    for k, v in later.items():
        dt, shape, raw = t[k]
        exp = oracle.convert(raw, "BF16", "F16") if dt is DType.BF16 else raw
        assert v.torch.reshape(-1).view(torch.uint8).cpu().numpy().tobytes() == exp, k
    fb.close()
    ld.close()


def test_kept_small_outputs_pin_a_small_chunk(tmp_path, rng):
    """auto_release outputs are carved from shared chunks (one cudaMalloc per
    chunk, not per key); outputs under CARVE_SMALL (norms, biases) come from
    their own CARVE_SMALL_CHUNK chunks, so a caller that keeps only those pins
    16 MiB, not a chunk of weights (ref device.py:191-214 releases per buffer)."""
    from paper_2505_23072_b200 import device

    t = {"w0": (DType.BF16, (2048, 1024), rng.integers(0, 256, 4 << 20, dtype=np.uint8).tobytes()),
         "n0": (DType.BF16, (1024,), rng.integers(0, 256, 2048, dtype=np.uint8).tobytes()),
         "w1": (DType.BF16, (1024, 1024), rng.integers(0, 256, 2 << 20, dtype=np.uint8).tobytes()),
         "b1": (DType.F32, (1024,), rng.integers(0, 256, 4096, dtype=np.uint8).tobytes())}
    p = _write(tmp_path, "m.safetensors", t)
    loader = SafeTensorsFileLoader(SingleGroup(), "host")
    loader.add_filenames({0: [p]})
    fb = loader.copy_files_to_device()
    got = {k: fb.get_tensor(k) for k in t}
    for k, (_, _, raw) in t.items():
        assert got[k].tobytes() == raw, k
    small = {k: got[k].torch.untyped_storage().nbytes() for k in ("n0", "b1")}
    big = {k: got[k].torch.untyped_storage().nbytes() for k in ("w0", "w1")}
    assert all(v == device.CARVE_SMALL_CHUNK for v in small.values()), small
    assert all(v >= (4 << 20) + (2 << 20) for v in big.values()), big  # the weights share one chunk
    kept = got["n0"].torch
    del got
    fb.close()
    loader.close()
    assert kept.untyped_storage().nbytes() == device.CARVE_SMALL_CHUNK
    assert kept.view(torch.uint8).cpu().numpy().tobytes() == t["n0"][2]


@pytest.mark.parametrize("residue", [1, 3, 481])
def test_realign_in_place_under_a_tight_device_cap(tmp_path, rng, residue, monkeypatch):
    """An odd header on the simdirect landing needs the realign; with a
    device_cap that holds the landing buffer but not a second copy, the loader
    repacks inside the landing buffer like the reference (device.py:466-534)
    instead of raising OutOfMemory — through small scratch windows here, so the
    overlapping (shift < window) and disjoint piece paths both run. Bytes are
    the file's (oracle)."""
    from paper_2505_23072_b200 import loader as loader_mod

    monkeypatch.setattr(loader_mod, "REPACK_WINDOW", 4096)
    t = {"a": (DType.F32, (3000,), rng.integers(0, 256, 12000, dtype=np.uint8).tobytes()),
         "b": (DType.BF16, (7, 4), rng.integers(0, 256, 56, dtype=np.uint8).tobytes()),  # writer-aligned begins
         "c": (DType.F64, (1001,), rng.integers(0, 256, 8008, dtype=np.uint8).tobytes()),
         "d": (DType.U8, (5,), rng.integers(0, 256, 5, dtype=np.uint8).tobytes())}
    p = _write(tmp_path, "odd.safetensors", t, pad=pad_for_body_residue(t, residue))
    probe = SafeTensorsFileLoader(SingleGroup(), "simdirect")
    probe.add_filenames({0: [p]})
    fb = probe.copy_files_to_device()
    cap = fb.transferred_buffer_bytes * 3 // 2  # room for the landing buffer, not for a second copy
    fb.close()
    probe.close()
    ld = SafeTensorsFileLoader(SingleGroup(), "simdirect", config=LoaderConfig(device_cap=cap, auto_release=False))
    ld.add_filenames({0: [p]})
    fb = ld.copy_files_to_device()
    for k, (_, _, raw) in t.items():
        assert fb.get_tensor(k).tobytes() == raw, k
    assert ld.pool.allocated_bytes <= cap
    fb.close()
    ld.close()
