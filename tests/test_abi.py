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
    assert C.sizeof(_native.hl_plan_stats) == 96


def test_version_and_conversion_table():
    lib = _native.load()
    assert lib.hl_abi_version() == 1 and b"sm_100a" in lib.hl_version()
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
