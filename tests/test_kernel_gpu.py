"""hl_gather (the sm_100a realign/shard/cast kernel) against the CPU oracle.

Bit-exact comparisons over the whole destination buffer (pre-filled with a
sentinel, so stray writes are caught too). The oracle is oracle/oracle_c.c
(numpy's conversion algorithm, pinned to the reference's outputs by
tests/golden/conv.npz).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle  # noqa: E402
from paper_2505_23072_b200 import _native, kernels  # noqa: E402
from paper_2505_23072_b200.errors import MisalignedDirectTransfer, UnsupportedConversion  # noqa: E402
from paper_2505_23072_b200.format import DType  # noqa: E402

pytestmark = pytest.mark.gpu

SIZES = [1, 1, 1, 2, 2, 4, 4, 8, 8, 2, 2, 4, 8]
CASTS = [(10, 9), (11, 9), (9, 11), (10, 11)]  # BF16->F16, F32->F16, F16->F32, BF16->F32
SENTINEL = 0xA5


def run_both(src: np.ndarray, dst_size: int, descs: list[tuple]):
    """descs: (src_off, dst_off, rows, row_elems, pitch, sdt, ddt) relative to
    the two buffers. Returns (gpu_bytes, oracle_bytes)."""
    dev = torch.device("cuda", 0)
    s = torch.from_numpy(src).to(dev)
    d = torch.full((dst_size + 64,), SENTINEL, dtype=torch.uint8, device=dev)
    kd = [(s.data_ptr() + so, d.data_ptr() + do, r, re, p, sd, dd) for so, do, r, re, p, sd, dd in descs]
    _native.gather(kd, torch.cuda.current_stream(dev).cuda_stream)
    got = d.cpu().numpy()
    lib = oracle.clib()
    exp = np.full(dst_size + 64, SENTINEL, dtype=np.uint8)
    sp, ep = src.ctypes.data, exp.ctypes.data
    for so, do, r, re, p, sd, dd in descs:
        if r and re:
            assert lib.oracle_gather(sp + so, ep + do, r, re, p, sd, dd) == 0
    return got, exp


def assert_same(got, exp):
    if not np.array_equal(got, exp):
        bad = np.nonzero(got != exp)[0]
        raise AssertionError(f"{bad.size} bytes differ; first at {bad[:8]}: got {got[bad[:8]]} exp {exp[bad[:8]]}")


@pytest.mark.parametrize("pair", CASTS)
@pytest.mark.parametrize("src_shift", [0, 1, 2, 3, 5, 8, 13])
def test_exhaustive_16bit_and_sampled_f32_casts(golden_conv, pair, src_shift):
    sdt, ddt = pair
    if sdt == 11:
        vals = golden_conv["f32_in"].astype("<u4")
        ref = golden_conv["f32_f16"]
    else:
        vals = golden_conv["all16"].astype("<u2")
        ref = {(10, 9): golden_conv["bf16_f16"], (9, 11): golden_conv["f16_f32"],
               (10, 11): golden_conv["bf16_f32"]}[pair]
    raw = vals.tobytes()
    src = np.zeros(len(raw) + 64, dtype=np.uint8)
    src[src_shift:src_shift + len(raw)] = np.frombuffer(raw, np.uint8)
    n = vals.size
    out_bytes = n * SIZES[ddt]
    got, exp = run_both(src, out_bytes, [(src_shift, 0, 1, n, len(raw), sdt, ddt)])
    assert_same(got, exp)
    # and the oracle itself equals the reference's outputs
    assert got[:out_bytes].tobytes() == ref.tobytes()


def _random_desc(rng, cursor_src, cursor_dst, src_cap):
    if rng.random() < 0.3:
        sdt, ddt = CASTS[int(rng.integers(0, 4))]
    else:
        sdt = int(rng.integers(0, 13))
        ddt = sdt
    ss, ds = SIZES[sdt], SIZES[ddt]
    rows = int(rng.choice([1, 1, 2, 3, 7, 16, 33]))
    row_elems = int(rng.choice([1, 2, 3, 5, 8, 15, 16, 64, 100, 257, 1024]))
    pad = int(rng.choice([0, 0, 1, 3, 8, 17]))  # strided (shard-like) rows when pad > 0
    pitch = (row_elems + pad) * ss
    src_off = cursor_src + int(rng.integers(0, 16))  # any byte: realign
    align = 16 if rng.random() < 0.7 else ds
    dst_off = -(-cursor_dst // align) * align
    need = src_off + (rows - 1) * pitch + row_elems * ss
    if need > src_cap:
        return None
    return (src_off, dst_off, rows, row_elems, pitch, sdt, ddt), need, dst_off + rows * row_elems * ds


@pytest.mark.parametrize("seed", range(6))
def test_random_batches(seed):
    rng = np.random.default_rng(seed)
    src_cap = 1 << 22
    src = rng.integers(0, 256, size=src_cap, dtype=np.uint8)
    descs, cs, cd = [], 0, 0
    for _ in range(int(rng.integers(50, 700))):  # > 560 exercises multi-launch batches
        r = _random_desc(rng, cs, cd, src_cap)
        if r is None:
            break
        d, cs, cd = r
        descs.append(d)
    got, exp = run_both(src, cd, descs)
    assert_same(got, exp)


@pytest.mark.parametrize("sdt,ddt", [(10, 10), (10, 9), (11, 9), (9, 11), (10, 11), (1, 1)])
@pytest.mark.parametrize("shift", [0, 1, 6, 13])
def test_large_contiguous(sdt, ddt, shift):
    rng = np.random.default_rng(7)
    n = (48 << 20) // SIZES[sdt] + 3  # ~48 MiB plus a ragged tail
    src = rng.integers(0, 256, size=n * SIZES[sdt] + 64, dtype=np.uint8)
    got, exp = run_both(src, n * SIZES[ddt], [(shift, 0, 1, n, n * SIZES[sdt], sdt, ddt)])
    assert_same(got, exp)


@pytest.mark.parametrize("dim", [0, 1, 2])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_shard_descriptors_match_reference_slicing(dim, world):
    rng = np.random.default_rng(dim * 10 + world)
    shape = (24, 40, 12)
    dt = DType.BF16
    raw = rng.integers(0, 256, size=int(np.prod(shape)) * 2, dtype=np.uint8)
    src = np.concatenate([np.zeros(3, np.uint8), raw, np.zeros(64, np.uint8)])
    dev = torch.device("cuda", 0)
    s = torch.from_numpy(src).to(dev)
    for rank in range(world):
        lo, hi = kernels.shard_bounds(shape[dim], world, rank)
        exp_shape, exp = oracle.slice_bytes(raw.tobytes(), "BF16", shape, dim, world, rank)
        out = torch.full((len(exp) + 32,), SENTINEL, dtype=torch.uint8, device=dev)
        kernels.run([kernels.shard_desc(s.data_ptr() + 3, shape, dim, lo, hi, out.data_ptr(), dt)], dev)
        got = out.cpu().numpy()
        assert got[: len(exp)].tobytes() == exp
        assert (got[len(exp):] == SENTINEL).all()


def test_errors_are_typed():
    dev = torch.device("cuda", 0)
    t = torch.zeros(64, dtype=torch.uint8, device=dev)
    p = t.data_ptr()
    with pytest.raises(UnsupportedConversion):
        _native.gather([(p, p + 32, 1, 2, 8, 12, 9)], 0)  # F64 -> F16
    with pytest.raises(MisalignedDirectTransfer):
        _native.gather([(p, p + 33, 1, 2, 8, 11, 11)], 0)  # F32 dst at odd address


def test_launch_counter_moves():
    dev = torch.device("cuda", 0)
    t = torch.zeros(1024, dtype=torch.uint8, device=dev)
    before = _native.kernel_launches()
    kernels.run([kernels.copy_desc(t.data_ptr(), t.data_ptr() + 512, 100, DType.F32)], dev)
    assert _native.kernel_launches() == before + 1


@pytest.mark.parametrize("sdt,ddt", [(10, 10), (1, 1), (10, 9), (11, 9), (9, 11), (10, 11), (7, 7)])
@pytest.mark.parametrize("shift", [0, 1, 5, 8, 15])
def test_long_rows_every_alignment(sdt, ddt, shift):
    """Row units (M_ROWS): many rows, source rows at varying misalignment
    (pitch not a multiple of 16), row lengths not multiples of 31 or 256
    vectors: the shifted (shuffle) path and its unit boundaries."""
    rng = np.random.default_rng(sdt * 100 + shift)
    ss, ds = SIZES[sdt], SIZES[ddt]
    row_elems = (16 // ds) * int(rng.choice([64, 100, 257, 513, 1030]))  # whole output vectors per row
    rows = int(rng.choice([1, 3, 37]))
    pitch = row_elems * ss + int(rng.choice([0, 3, 8, 24]))
    src = rng.integers(0, 256, size=shift + rows * pitch + 64, dtype=np.uint8)
    got, exp = run_both(src, rows * row_elems * ds, [(shift, 0, rows, row_elems, pitch, sdt, ddt)])
    assert_same(got, exp)


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("dim", [0, 1, 2])
@pytest.mark.parametrize("cast", [None, "F16"])
def test_nccl_plane_owner_pack(world, dim, cast):
    """The NCCL data plane's device work: the owner packs every rank's slice
    (cast fused) with one hl_gather launch; parts equal the reference slicing."""
    from paper_2505_23072_b200.collective import pack_parts, partition
    from paper_2505_23072_b200.format import TensorMetadata

    rng = np.random.default_rng(world * 10 + dim)
    shape = (24, 40, 16)
    raw = rng.integers(0, 256, size=int(np.prod(shape)) * 2, dtype=np.uint8)
    dev = torch.device("cuda", 0)
    s = torch.from_numpy(np.concatenate([np.zeros(5, np.uint8), raw, np.zeros(64, np.uint8)])).to(dev)
    spec = partition(TensorMetadata("w", DType.BF16, shape, (0, raw.size)), dim, world)
    out_dt = DType.F16 if cast else DType.BF16
    own = world - 1
    own_out = torch.empty(int(np.prod(spec.part_shapes[own])) * 2, dtype=torch.uint8, device=dev)
    launches = _native.kernel_launches()
    parts = pack_parts(spec, s.data_ptr() + 5, DType.BF16, out_dt, own, own_out, dev)
    assert _native.kernel_launches() - launches <= 3  # one per kernel variant present
    src_bytes = oracle.convert(raw.tobytes(), "BF16", "F16") if cast else raw.tobytes()
    for r in range(world):
        _, exp = oracle.slice_bytes(src_bytes, out_dt.value, shape, dim, world, r)
        assert parts[r].cpu().numpy().tobytes() == exp, (r, dim, world, cast)
    assert parts[own].data_ptr() == own_out.data_ptr()
    # with the source bytes at hand, a part that is one contiguous source range (dim 0, no
    # cast) is sent straight from the source: no pack copy, same bytes
    parts = pack_parts(spec, s.data_ptr() + 5, DType.BF16, out_dt, own, own_out, dev, src_bytes=s[5:5 + raw.size])
    for r in range(world):
        _, exp = oracle.slice_bytes(src_bytes, out_dt.value, shape, dim, world, r)
        assert parts[r].cpu().numpy().tobytes() == exp, ("direct", r, dim, world, cast)
        in_source = s.data_ptr() <= parts[r].data_ptr() < s.data_ptr() + s.numel()
        assert in_source == (r != own and dim == 0 and not cast), (r, dim, cast)


@pytest.mark.parametrize("seed", range(4))
def test_many_multi_unit_tensors(seed):
    """Hundreds of contiguous tensors of 1-4 TMA units (8-16 KiB source units)
    each, every kind, random source shifts and 16-byte aligned destinations:
    the bulk and staged kernels walk descriptor boundaries inside their stage
    rings (each CTA sees many units; stages wrap many times)."""
    rng = np.random.default_rng(100 + seed)
    kinds = [(10, 10), (1, 1), (10, 9), (11, 9), (9, 11), (10, 11)]
    src_cap = 48 << 20
    src = rng.integers(0, 256, size=src_cap, dtype=np.uint8)
    descs, cs, cd = [], 0, 0
    for _ in range(900):  # > 500: several launches per kernel
        sdt, ddt = kinds[int(rng.integers(0, len(kinds)))]
        n = int(rng.integers(1, 4 * 16384 // SIZES[sdt]))
        shift = int(rng.integers(0, 16)) if rng.random() < 0.5 else 0
        so = cs + shift
        if so + n * SIZES[sdt] > src_cap:
            break
        descs.append((so, cd, 1, n, n * SIZES[sdt], sdt, ddt))
        cs = (so + n * SIZES[sdt] + 15) & ~15
        cd = (cd + n * SIZES[ddt] + 15) & ~15
    got, exp = run_both(src, cd, descs)
    assert_same(got, exp)


def test_no_tma_flag_gives_identical_bytes():
    """hl_gather_ex(..., HL_GATHER_NO_TMA) (the peer-pull path) routes contiguous
    copies/casts to the LDG/STG kernels: same bytes as the TMA kernels."""
    rng = np.random.default_rng(5)
    src = rng.integers(0, 256, size=8 << 20, dtype=np.uint8)
    descs, cs, cd = [], 0, 0
    for sdt, ddt in [(10, 10), (1, 1), (10, 9), (11, 9), (9, 11), (10, 11)] * 4:
        n = int(rng.integers(1, 100_000))
        so = cs + int(rng.integers(0, 16))
        descs.append((so, cd, 1, n, n * SIZES[sdt], sdt, ddt))
        cs = (so + n * SIZES[sdt] + 15) & ~15
        cd = (cd + n * SIZES[ddt] + 15) & ~15
    dev = torch.device("cuda", 0)
    s = torch.from_numpy(src).to(dev)
    outs = []
    for flags in (0, _native.GATHER_NO_TMA):
        d = torch.full((cd + 64,), SENTINEL, dtype=torch.uint8, device=dev)
        kd = [(s.data_ptr() + so, d.data_ptr() + do, r, re, p, sd, dd) for so, do, r, re, p, sd, dd in descs]
        _native.gather(kd, torch.cuda.current_stream(dev).cuda_stream, flags)
        outs.append(d.cpu().numpy())
    assert_same(outs[1], outs[0])
    _, exp = run_both(src, cd, descs)
    assert_same(outs[0], exp)


TILE_KINDS = [(10, 10), (1, 1), (11, 11), (7, 7), (10, 9), (11, 9), (9, 11), (10, 11)]


@pytest.mark.parametrize("sdt,ddt", TILE_KINDS)
@pytest.mark.parametrize("seed", range(5))
def test_column_shard_tiles(sdt, ddt, seed):
    """Column shards (rows > 1, pitch > row): the 2-D tensor-map TMA kernels
    (tile_copy_kernel / tile_cast_kernel) — box edges inside and at the end of
    rows, ragged last boxes, >256 rows, every rank of W = 2/3/8 (source
    offsets at every element position), plus the narrow-row / odd-width cases
    that stay on the warp kernels; all against the oracle, with sentinels."""
    rng = np.random.default_rng(1000 * seed + 10 * sdt + ddt)
    ss, ds = SIZES[sdt], SIZES[ddt]
    world = int(rng.choice([2, 3, 8]))
    rows = int(rng.choice([2, 33, 257, 600]))
    cols = int(rng.choice([64, 96, 1000, 1024, 4096, 2304])) * max(1, 8 // ss)
    lead = int(rng.choice([0, ss, 16]))
    src = rng.integers(0, 256, size=lead + rows * cols * ss + 64, dtype=np.uint8)
    descs, cd = [], 0
    for r in range(world):
        lo, hi = kernels.shard_bounds(cols, world, r)
        descs.append((lead + lo * ss, cd, rows, hi - lo, cols * ss, sdt, ddt))
        cd = (cd + rows * (hi - lo) * ds + 15) & ~15
    got, exp = run_both(src, cd, descs)
    assert_same(got, exp)


@pytest.mark.parametrize("shape,dt,cast", [((4096, 8192), 10, None), ((4096, 8192), 10, 9),
                                           ((2048, 3072), 11, 9), ((1024, 5120), 10, 11)])
def test_tp8_column_shards_large(shape, dt, cast):
    """70B-sized column shards (TP=8 along dim 1): the owner-pack batch of the
    NCCL plane and the C4/C5 workload shape, bit-exact."""
    rng = np.random.default_rng(shape[1] + dt)
    rows, cols = shape
    ss = SIZES[dt]
    ddt = cast or dt
    src = rng.integers(0, 256, size=rows * cols * ss + 64, dtype=np.uint8)
    descs, cd = [], 0
    for r in range(8):
        lo, hi = kernels.shard_bounds(cols, 8, r)
        descs.append((lo * ss, cd, rows, hi - lo, cols * ss, dt, ddt))
        cd = (cd + rows * (hi - lo) * SIZES[ddt] + 15) & ~15
    got, exp = run_both(src, cd, descs)
    assert_same(got, exp)


def test_many_column_shards_span_tile_launches():
    """More column-shard descriptors than one tile launch carries (96): the
    launch split and the per-descriptor unit walk."""
    rng = np.random.default_rng(77)
    src = rng.integers(0, 256, size=16 << 20, dtype=np.uint8)
    descs, cs, cd = [], 0, 0
    for i in range(250):
        rows = int(rng.integers(2, 40))
        cols = 8 * int(rng.integers(8, 200))
        seg = 8 * int(rng.integers(4, cols // 8 + 1))
        lo = 8 * int(rng.integers(0, (cols - seg) // 8 + 1))
        sdt, ddt = [(10, 10), (10, 9), (1, 1)][i % 3]
        ss = SIZES[sdt]
        if cs + rows * cols * ss + 64 > src.size:
            break
        descs.append((cs + lo * ss, cd, rows, seg, cols * ss, sdt, ddt))
        cs = (cs + rows * cols * ss + 15) & ~15
        cd = (cd + rows * seg * SIZES[ddt] + 15) & ~15
    got, exp = run_both(src, cd, descs)
    assert_same(got, exp)


@pytest.mark.parametrize("world", [7, 8])
def test_interleaved_shard_groups_across_launches(world):
    """A tensor's W column shards form one interleave group (tile_unit: unit u
    of the group is unit u / W of shard u % W), so the grid streams the same
    rows of every shard together. 40 tensors x W shards is more than one tile
    launch carries (96): groups never straddle a launch (W=7 leaves a gap);
    uneven splits give shards of different widths (partial groups); casts and
    raw copies mixed. Against the oracle, with sentinels."""
    rng = np.random.default_rng(500 + world)
    src = rng.integers(0, 256, size=48 << 20, dtype=np.uint8)
    descs, cs, cd = [], 0, 0
    for i in range(40):
        rows = int(rng.choice([16, 40, 300]))
        cols = 8 * world * int(rng.integers(4, 40)) + (8 * int(rng.integers(0, world)) if i % 4 == 3 else 0)
        sdt, ddt = [(10, 10), (10, 9), (11, 9), (1, 1)][i % 4]
        ss = SIZES[sdt]
        if cs + rows * cols * ss + 64 > src.size:
            break
        for r in range(world):
            lo, hi = kernels.shard_bounds(cols, world, r)
            descs.append((cs + lo * ss, cd, rows, hi - lo, cols * ss, sdt, ddt))
            cd = (cd + rows * (hi - lo) * SIZES[ddt] + 15) & ~15
        cs = (cs + rows * cols * ss + 15) & ~15
    assert len(descs) > 96
    got, exp = run_both(src, cd, descs)
    assert_same(got, exp)


@pytest.mark.parametrize("rows,cols,dt,world,lead", [
    (4096, 4096, 10, 8, 0),      # 7B o_proj at TP=8: 1 KiB of every 8 KiB row per shard
    (1024, 28672, 10, 8, 0),     # 70B down_proj rows (56 KiB) span several 16 KiB chunks
    (300, 1000, 10, 8, 0),       # uneven widths (remainder columns), 16-byte aligned
    (257, 4096, 11, 4, 16),      # f32, W=4, tensor not at the buffer start
    (64, 2304, 1, 16, 0),        # u8, W=16: the most shards a split descriptor carries
    (129, 96, 10, 2, 0),         # pitch smaller than a bulk chunk: one chunk holds many rows
])
def test_row_split_owner_pack(rows, cols, dt, world, lead):
    """All W column shards of one tensor in a row (the NCCL plane's owner pack),
    between unrelated descriptors: bit-exact against the oracle with sentinels
    around every output (interleaved tile groups; uneven widths on the row
    kernel)."""
    rng = np.random.default_rng(rows * 7 + cols + world)
    es = SIZES[dt]
    src = rng.integers(0, 256, size=lead + rows * cols * es + 4096 + 64, dtype=np.uint8)
    descs, cd = [(lead + rows * cols * es, 0, 1, 100, 100 * es, dt, dt)], ((100 * es + 15) & ~15) + 16
    for r in range(world):
        lo, hi = kernels.shard_bounds(cols, world, r)
        descs.append((lead + lo * es, cd, rows, hi - lo, cols * es, dt, dt))
        cd = (cd + rows * (hi - lo) * es + 16 + 15) & ~15  # a sentinel gap after every shard
    descs.append((lead + 64 * es, cd, 3, 40, 200 * es, dt, dt))
    cd += 3 * 40 * es + 64
    l0 = _native.kernel_launches()
    got, exp = run_both(src, cd, descs)
    assert _native.kernel_launches() > l0
    assert_same(got, exp)


def test_launch_timing_pairs_every_call():
    """hl_gather_timing / hl_gather_timings (bench.py's roofline timer): one
    event pair per hl_gather call while enabled, positive durations in call
    order, nothing recorded while disabled."""
    dev = torch.device("cuda", 0)
    src = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
    dst = torch.empty_like(src)
    d = kernels.copy_desc(src.data_ptr(), dst.data_ptr(), src.numel(), DType.U8)
    _native.gather_timing(False)
    kernels.run([d], dev)
    assert _native.gather_timings() == []
    _native.gather_timing(True)
    try:
        for _ in range(3):
            kernels.run([d], dev)
        ms = _native.gather_timings()
        assert len(ms) == 3 and all(t > 0 for t in ms), ms
        assert _native.gather_timings() == []  # fetched pairs are forgotten
    finally:
        _native.gather_timing(False)
