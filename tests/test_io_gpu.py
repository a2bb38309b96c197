"""The bulk file -> HBM engine (hl_execute_plan) in every I/O mode."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2505_23072_b200 import _native  # noqa: E402
from paper_2505_23072_b200.errors import IoError  # noqa: E402

pytestmark = pytest.mark.gpu

MODES = ["buffered", "direct", "auto", "cufile", "mmap", "auto-pin"]


@pytest.fixture(scope="module")
def blob(tmp_path_factory):
    rng = np.random.default_rng(11)
    data = rng.integers(0, 256, size=(37 << 20) + 4093, dtype=np.uint8)
    p = tmp_path_factory.mktemp("io") / "blob.bin"
    p.write_bytes(data.tobytes())
    return p, data


@pytest.mark.parametrize("mode", MODES)
def test_ranges_land_exactly(blob, mode):
    path, data = blob
    if mode == "auto-pin":  # resident chunks DMA'd from the page cache in place (HL_CFG_AUTO_PIN_CACHE)
        eng = _native.IoEngine(0, workers=4, chunk_bytes=1 << 20, io_mode="auto", flags=_native.HL_CFG_AUTO_PIN_CACHE)
        path.read_bytes()  # resident
    else:
        eng = _native.IoEngine(0, workers=4, chunk_bytes=1 << 20, io_mode=mode)
    rng = np.random.default_rng(3)
    ranges = [(0, data.size), (1, 4095), (4096, 8192), (13281, (5 << 20) + 7), (data.size - 9, 9)]
    for _ in range(6):
        off = int(rng.integers(0, data.size - 1))
        ranges.append((off, int(rng.integers(1, min(6 << 20, data.size - off)))))
    total = sum(n for _, n in ranges)
    dst = torch.zeros(total + 64, dtype=torch.uint8, device="cuda")
    blocks, cur = [], 0
    for i, (off, n) in enumerate(ranges):
        blocks.append((0, i, off, n, dst.data_ptr() + cur))
        cur += n
    st = eng.execute([str(path)], blocks)
    assert st["bytes"] == total
    got = dst.cpu().numpy()
    cur = 0
    for off, n in ranges:
        assert np.array_equal(got[cur:cur + n], data[off:off + n]), (mode, off, n)
        cur += n
    assert st["io_modes"], st
    if mode == "auto-pin" and st["mmap_bytes"]:
        # resident chunks went straight from the page cache (hosts whose kernel refuses to pin
        # file pages — cudaHostRegister EINVAL, profiles/r02_host_register_probe.txt — fall back
        # to the ring, which the byte check above covers)
        assert "mmap" in st["io_modes"], st
    eng.close()


def test_read_past_eof_is_io_error(blob):
    path, data = blob
    eng = _native.IoEngine(0, workers=2, chunk_bytes=1 << 20, io_mode="buffered")
    dst = torch.zeros(8192, dtype=torch.uint8, device="cuda")
    with pytest.raises(IoError):
        eng.execute([str(path)], [(0, 0, data.size - 10, 100, dst.data_ptr())])
    with pytest.raises(IoError):
        eng.execute(["/nonexistent/file"], [(0, 0, 0, 10, dst.data_ptr())])


def test_residency_and_drop_cache(blob):
    path, data = blob
    _ = path.read_bytes()  # warm
    assert _native.file_residency(str(path)) > 0.5
    _native.drop_cache(str(path))
    assert _native.file_residency(str(path)) < 0.5
    # auto mode now reads with O_DIRECT and still lands the right bytes
    eng = _native.IoEngine(0, workers=4, chunk_bytes=1 << 20, io_mode="auto")
    dst = torch.zeros(data.size, dtype=torch.uint8, device="cuda")
    st = eng.execute([str(path)], [(0, 0, 0, data.size, dst.data_ptr())])
    assert "direct" in st["io_modes"] or "buffered" in st["io_modes"]
    assert np.array_equal(dst.cpu().numpy(), data)


def test_forced_cufile_compat_mode_in_subprocess(blob, tmp_path):
    """cuFile without nvidia-fs (compat mode) is not used by default; this
    probes it in a child process under a timeout and records what happens."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    path, data = blob
    code = (
        "import sys, torch, numpy as np; sys.path.insert(0, %r)\n"
        "from paper_2505_23072_b200 import _native\n"
        "eng = _native.IoEngine(0, workers=1, chunk_bytes=1<<20, io_mode='cufile')\n"
        "d = torch.zeros(%d, dtype=torch.uint8, device='cuda')\n"
        "st = eng.execute([%r], [(0, 0, 0, %d, d.data_ptr())])\n"
        "print('MODES', st['io_modes'])\n"
        "ok = np.array_equal(d.cpu().numpy(), np.fromfile(%r, dtype=np.uint8)[:%d])\n"
        "print('EQUAL', ok)\n" % (str(ROOT), 4 << 20, str(path), 4 << 20, str(path), 4 << 20))
    env = dict(os.environ, HL_FORCE_CUFILE="1")
    try:
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=30)
    except subprocess.TimeoutExpired:
        pytest.xfail("cuFile compat mode (no nvidia-fs) hangs in cuFileRead on this host")
    if r.returncode != 0:
        pytest.xfail(f"cuFile compat mode unavailable: {r.stderr.strip().splitlines()[-1:]}")
    assert "EQUAL True" in r.stdout, r.stdout + r.stderr


def test_auto_mode_is_per_chunk_hybrid(blob):
    """AUTO reads what the page cache holds (mincore probe) and the rest with
    O_DIRECT, per chunk: a half-cached file uses both paths and lands exactly."""
    import os
    import time

    path, data = blob
    _native.drop_cache(str(path))
    # warm the first half only, with WILLNEED: a read() would leave readahead
    # markers whose async readahead pulls the cold half in ahead of the probes
    fd = os.open(str(path), os.O_RDONLY)
    os.posix_fadvise(fd, 0, data.size // 2, os.POSIX_FADV_WILLNEED)
    os.close(fd)
    t0 = time.time()
    while _native.file_residency(str(path)) < 0.45 and time.time() - t0 < 5:
        time.sleep(0.05)
    eng = _native.IoEngine(0, workers=4, chunk_bytes=1 << 20, io_mode="auto")
    dst = torch.zeros(data.size, dtype=torch.uint8, device="cuda")
    st = eng.execute([str(path)], [(0, 0, 0, data.size, dst.data_ptr())])
    assert st["buffered_bytes"] > 0 and st["direct_bytes"] > 0, st
    assert st["buffered_bytes"] + st["direct_bytes"] == data.size
    assert np.array_equal(dst.cpu().numpy(), data)
    # unaligned ranges through the hybrid path
    _native.drop_cache(str(path))
    rng = np.random.default_rng(9)
    for _ in range(8):
        off = int(rng.integers(0, data.size - 1))
        n = int(rng.integers(1, min(3 << 20, data.size - off)))
        d2 = torch.zeros(n + 16, dtype=torch.uint8, device="cuda")
        eng.execute([str(path)], [(0, 0, off, n, d2.data_ptr())])
        assert np.array_equal(d2.cpu().numpy()[:n], data[off:off + n])


def test_engine_writes_wait_for_the_callers_stream(blob):
    """Write-after-read guard (hl_execute_plan_after): a copy queued on the
    current stream behind a long spin still reads the OLD bytes of a buffer
    the engine is asked to overwrite right away."""
    path, data = blob
    n = 8 << 20
    eng = _native.IoEngine(0, workers=4, chunk_bytes=1 << 20, io_mode="buffered")
    old = torch.full((n,), 7, dtype=torch.uint8, device="cuda")
    out = torch.empty_like(old)
    torch.cuda.synchronize()
    torch.cuda._sleep(400_000_000)  # ~0.2 s of spinning on the current stream
    out.copy_(old)  # queued behind the spin
    eng.execute([str(path)], [(0, 0, 0, n, old.data_ptr())],
                after_stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert bool((out == 7).all()), "the engine overwrote bytes a queued kernel had not read yet"
    assert np.array_equal(old.cpu().numpy(), data[:n])
    eng.close()


def test_worker_team_is_persistent_and_pinned(blob):
    """The engine's team is spawned once per context (no threads per plan)
    and every team thread runs on the context's CPUs (ref transfer.py:274-293)."""
    import os

    path, data = blob
    eng = _native.IoEngine(0, workers=3, chunk_bytes=1 << 20, io_mode="buffered")
    dst = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")

    def team():
        out = {}
        for tid in os.listdir("/proc/self/task"):
            try:
                name = open(f"/proc/self/task/{tid}/comm").read().strip()
            except OSError:
                continue
            if name.startswith("hl-io-0-"):
                out[int(tid)] = os.sched_getaffinity(int(tid))
        return out

    before = {t for t in team()}
    eng.execute([str(path)], [(0, 0, 0, 4 << 20, dst.data_ptr())])
    first = team()
    eng.execute([str(path)], [(0, 0, 0, 4 << 20, dst.data_ptr())])
    second = team()
    new = {t: a for t, a in first.items() if t not in before}
    assert len(new) == 3 and set(second) == set(first)
    cpus = eng.cpus()
    if cpus:
        assert all(a == set(cpus) for a in new.values())
    eng.close()
    assert not set(new) & set(team())  # joined on close


def test_cold_plans_run_on_the_cold_team(blob):
    """A plan that is mostly O_DIRECT reads (direct mode, or auto with the file
    dropped from the page cache) runs on the larger cold-reader team; a resident
    one keeps the configured team. Bytes are exact either way."""
    path, data = blob
    n = 32 << 20
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    eng = _native.IoEngine(0, workers=4, chunk_bytes=1 << 20, io_mode="auto")
    path.read_bytes()
    warm = eng.execute([str(path)], [(0, 0, 0, n, dst.data_ptr())], after_stream=0)
    assert warm["workers"] == 4 and np.array_equal(dst.cpu().numpy(), data[:n])
    _native.drop_cache(str(path))
    dst.zero_()
    cold = eng.execute([str(path)], [(0, 0, 0, n, dst.data_ptr())], after_stream=0)
    # io_uring threads with many reads in flight, or (io_uring unavailable) the larger team
    assert "direct" in cold["io_modes"], cold
    assert "io_uring" in cold["io_modes"] or cold["workers"] > 4, cold
    assert np.array_equal(dst.cpu().numpy(), data[:n])
    eng.close()


@pytest.mark.parametrize("uring", ["1", "0"])
def test_cold_reader_paths_give_identical_bytes(blob, monkeypatch, uring):
    """Cold plans read through io_uring (HL_COLD_URING, default on) or the
    blocking reader team (HL_COLD_URING=0): ragged ranges at odd offsets,
    the file's last bytes (a short O_DIRECT read at EOF), a partly resident
    file, tiny rings (reads wait on slot DMAs), and the async tail — the same
    bytes either way."""
    monkeypatch.setenv("HL_COLD_URING", uring)
    monkeypatch.setenv("HL_URING_DEPTH", "5")
    path, data = blob
    rng = np.random.default_rng(11)
    ranges = [(0, 3 << 20), (13281, (5 << 20) + 7), (data.size - 9, 9), (4095, 2)]
    for _ in range(8):
        off = int(rng.integers(0, data.size - 1))
        ranges.append((off, int(rng.integers(1, min(7 << 20, data.size - off)))))
    total = sum(n for _, n in ranges)
    s = torch.cuda.current_stream().cuda_stream
    eng = _native.IoEngine(0, workers=3, chunk_bytes=1 << 20, slots_per_worker=2, io_mode="auto")
    for resident in (False, True, "half"):
        _native.drop_cache(str(path))
        if resident is True:
            path.read_bytes()
        elif resident == "half":
            with open(path, "rb") as f:
                f.read(data.size // 2)
        dst = torch.zeros(total + 64, dtype=torch.uint8, device="cuda")
        blocks, cur = [], 0
        for i, (off, n) in enumerate(ranges):
            blocks.append((0, i, off, n, dst.data_ptr() + cur))
            cur += n
        st = eng.execute([str(path)], blocks, after_stream=s, async_tail=True)
        got = dst.cpu().numpy()  # after the stream: the copies' completion was handed to it
        cur = 0
        for off, n in ranges:
            assert np.array_equal(got[cur:cur + n], data[off:off + n]), (uring, resident, off, n)
            cur += n
        if resident is False:
            assert ("io_uring" in st["io_modes"]) == (uring == "1"), st
    eng.close()


def test_async_plans_hand_completion_to_the_stream(blob):
    """hl_execute_plan_async returns once the copies are submitted; work
    enqueued on the stream afterwards (here a clone, no host sync in between)
    sees every byte, also across back-to-back plans that reuse the ring slots
    while earlier copies may still be in flight."""
    path, data = blob
    n = 12 << 20
    eng = _native.IoEngine(0, workers=3, chunk_bytes=1 << 20, io_mode="buffered")
    s = torch.cuda.current_stream().cuda_stream
    outs = []
    for i in range(6):
        off = (i * 5 << 20) % (data.size - n)
        dst = torch.empty(n, dtype=torch.uint8, device="cuda")
        eng.execute([str(path)], [(0, 0, off, n, dst.data_ptr())], after_stream=s, async_tail=True)
        outs.append((off, dst.clone()))  # enqueued behind the plan's copies
        del dst  # stream-ordered free: must not be recycled under an in-flight copy
    torch.cuda.synchronize()
    for off, got in outs:
        assert np.array_equal(got.cpu().numpy(), data[off:off + n]), off
    eng.close()


def test_small_warm_plans_run_on_half_a_large_team(blob, monkeypatch):
    """A warm plan under 2 GiB on a team of >= 8 runs on half of it (its copy
    engine is the bound; fewer concurrent page-cache copies leave it more host
    memory bandwidth); $HL_SMALL_TEAM overrides; bytes exact either way."""
    path, data = blob
    n = 24 << 20
    path.read_bytes()
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    eng = _native.IoEngine(0, workers=8, chunk_bytes=1 << 20, io_mode="auto")
    st = eng.execute([str(path)], [(0, 0, 0, n, dst.data_ptr())], after_stream=0)
    assert st["workers"] == 4 and np.array_equal(dst.cpu().numpy(), data[:n]), st
    monkeypatch.setenv("HL_SMALL_TEAM", "8")
    dst.zero_()
    st = eng.execute([str(path)], [(0, 0, 0, n, dst.data_ptr())], after_stream=0)
    assert st["workers"] == 8 and np.array_equal(dst.cpu().numpy(), data[:n]), st
    eng.close()
