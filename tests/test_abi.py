"""The C ABI: libhbmload.so loads on a GPU-less host, exports every symbol
include/hbmload.h declares, struct layouts agree with the ctypes mirror,
and without a device it fails loudly (typed error, no CPU fallback)."""

from __future__ import annotations

import ctypes as C
import re
import subprocess
import sys

import pytest

from conftest import ROOT
from oracle import oracle
from paper_2505_23072_b200 import _native
from paper_2505_23072_b200.errors import DeviceError, NativeUnavailable

HEADER = (ROOT / "include" / "hbmload.h").read_text()


def declared():
    body = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    return sorted(set(re.findall(r"\b(hl_[a-z_]+)\s*\(", body)))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    names = declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_native.SIGNATURES), set(names) ^ set(_native.SIGNATURES)
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\sT {n}$", nm, re.M), n


def test_struct_sizes_match_header_layout():
    assert C.sizeof(_native.hl_desc) == 48
    assert C.sizeof(_native.hl_block) == 32
    assert C.sizeof(_native.hl_config) == 32
    assert C.sizeof(_native.hl_plan_stats) == 120


def test_version_and_conversion_table():
    lib = _native.load()
    assert lib.hl_abi_version() == 2 and b"sm_100a" in lib.hl_version()
    assert lib.hl_gather_max_batch() >= 256
    for s in range(13):
        for d in range(13):
            exp = 1 if (s == d or (s, d) in {(10, 9), (11, 9), (9, 11), (10, 11)}) else 0
            assert lib.hl_conversion_supported(s, d) == exp
            if oracle.clib() is not None:
                assert oracle.clib().oracle_conversion_supported(s, d) == exp
    assert lib.hl_conversion_supported(13, 0) == 0


def test_fails_loudly_without_a_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(DeviceError):
        _native.IoEngine(0)
    from paper_2505_23072_b200 import SafeTensorsFileLoader, SingleGroup

    with pytest.raises(NativeUnavailable):
        SafeTensorsFileLoader(SingleGroup(), "host")


def test_sm100a_cubin_and_kernel_symbols():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "row_kernel" in sass and "generic_kernel" in sass
    assert "LDG.E.128" in sass or "LDG.E.ENL2.128" in sass or re.search(r"LDG\.E\S*\.128", sass)
    assert re.search(r"STG\.E\S*\.128", sass)
    # the TMA kernels: bulk copies both ways and mbarrier transaction counting
    assert "bulk_kernel" in sass and "staged_kernel" in sass
    assert "UBLKCP.S.G" in sass and "UBLKCP.G.S" in sass and "SYNCS.ARRIVE.TRANS64" in sass


def test_product_never_imports_the_oracle():
    pkg = ROOT / "paper_2505_23072_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f


def test_missing_library_is_an_error(tmp_path):
    code = ("import paper_2505_23072_b200._native as n; from pathlib import Path\n"
            "n.LIB_PATH = Path('/nonexistent/libhbmload.so')\n"
            "try:\n  n.load()\nexcept Exception as e:\n  print(type(e).__name__)\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT).stdout
    assert "NativeUnavailable" in out


CUDA = "/usr/local/cuda"


def _build_c_smoke(out_dir):
    exe = out_dir / "abi_smoke"
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-std=c11", f"-I{ROOT / 'include'}", f"-I{CUDA}/include",
           str(ROOT / "tests" / "c" / "abi_smoke.c"), "-o", str(exe),
           f"-L{_native.LIB_PATH.parent}", "-lhbmload", f"-L{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{_native.LIB_PATH.parent}:{CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_builds_against_the_header(tmp_path):
    """A plain C11 host (no Python, no torch) compiles and links against
    include/hbmload.h + libhbmload.so: the boundary is self-contained."""
    _build_c_smoke(tmp_path)


@pytest.mark.gpu
def test_c_program_loads_realigns_casts_and_shards(tmp_path, rng):
    import numpy as np

    exe = _build_c_smoke(tmp_path)
    raw = rng.integers(0, 256, size=(1 << 20) + 37, dtype=np.uint8)
    src = tmp_path / "blob.bin"
    src.write_bytes(raw.tobytes())
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), str(src), str(out)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "error path ok" in r.stdout
    launches = int(re.search(r"launches (\d+)", r.stdout).group(1))
    assert 1 <= launches <= 3  # one per (conversion kind, kernel variant) present in the batch
    got = out.read_bytes()
    nb, nc, rows, cols, lo, hi = 100003, 65536, 37, 300, 100, 200
    b = raw[3:3 + nb].tobytes()
    c = oracle.convert(raw[16:16 + 2 * nc].tobytes(), "BF16", "F16")
    d = raw[64:64 + rows * cols * 2].reshape(rows, cols * 2)[:, lo * 2:hi * 2].tobytes()
    assert got[:nb] == b
    assert got[nb:nb + len(c)] == c
    assert got[nb + len(c):] == d
