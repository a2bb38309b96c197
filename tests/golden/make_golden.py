"""Generate the golden fixtures from the REFERENCE implementation itself.

Runs only in the build container, where /root/reference exists; the outputs
are committed so the GPU box (which has no /root/reference) can check
against them. Re-run:  python tests/golden/make_golden.py

Outputs (tests/golden/):
  conv.npz         reference conversions (aggload.device._convert_elements,
                   device.py:310-320): exhaustive BF16->F16, BF16->F32,
                   F16->F32 over all 65,536 patterns; F32->F16 over 196,608
                   structured + random patterns. Also numpy.__version__.
  corpora/*.safetensors + expect.json
                   small random corpora (all 13 dtypes, odd header residues)
                   and, per (backend, world, dim), what the reference LOADER
                   returns on every rank for every key: kind (shard/full),
                   shape and sha256 of the bytes (aggload.loader with thread
                   ranks, exactly like test_acceptance.py:88-159), plus the
                   simdirect relocation table (align_fix dev_offsets).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import threading
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

from aggload.collective import ProcessGroup  # noqa: E402  (reference code, read-only import)
from aggload.device import _convert_elements  # noqa: E402
from aggload.format import DType, write_file  # noqa: E402
from aggload.loader import LoaderConfig, SafeTensorsFileLoader  # noqa: E402
from aggload.transfer import NumaNode, Topology  # noqa: E402

DIMS = [0, 1, 1, 2, 2, 3, 3, 4, 5, 7, 8, 13, 16, 64]


def conv_vectors() -> None:
    all16 = np.arange(65536, dtype=np.uint32).astype("<u2")
    raw16 = all16.tobytes()
    bf16_f16 = np.frombuffer(_convert_elements(np.frombuffer(raw16, np.uint8), DType.BF16, DType.F16), "<u2")
    bf16_f32 = np.frombuffer(_convert_elements(np.frombuffer(raw16, np.uint8), DType.BF16, DType.F32), "<u4")
    f16_f32 = np.frombuffer(_convert_elements(np.frombuffer(raw16, np.uint8), DType.F16, DType.F32), "<u4")
    rng = np.random.default_rng(0xF32F16)
    # every exponent x sign x {boundary mantissas}, plus uniform random bits
    exps = np.arange(256, dtype=np.uint32) << 23
    mants = np.array([0, 1, 0x1000, 0xFFF, 0x1FFF, 0x2000, 0x3000, 0x3FFF, 0x7FF, 0x800, 0x400000,
                      0x7FFFFF, 0x7FE000, 0x7FF000, 0x001001, 0x2001], dtype=np.uint32)
    structured = (exps[:, None] | mants[None, :]).reshape(-1)
    structured = np.concatenate([structured, structured | 0x80000000])
    rand = rng.integers(0, 2**32, size=196608 - structured.size, dtype=np.uint64).astype(np.uint32)
    f32 = np.concatenate([structured, rand]).astype("<u4")
    f32_f16 = np.frombuffer(_convert_elements(np.frombuffer(f32.tobytes(), np.uint8), DType.F32, DType.F16), "<u2")
    np.savez_compressed(HERE / "conv.npz", all16=all16, bf16_f16=bf16_f16, bf16_f32=bf16_f32, f16_f32=f16_f32,
                        f32_in=f32, f32_f16=f32_f16, numpy_version=np.array(np.__version__))


def random_tensors(rng, n, prefix):
    dts = list(DType)
    out = {}
    for i in range(n):
        dt = dts[int(rng.integers(0, len(dts)))]
        rank = int(rng.integers(0, 5))
        shape = tuple(int(rng.choice(DIMS)) for _ in range(rank))
        while int(np.prod(shape, dtype=np.int64)) > 4096:
            shape = tuple(min(d, 4) for d in shape)
        nb = int(np.prod(shape, dtype=np.int64)) * dt.size_bytes if shape else dt.size_bytes
        out[f"{prefix}{i}"] = (dt, shape, rng.integers(0, 256, size=nb, dtype=np.uint8).tobytes())
    return out


def pad_for_residue(tensors, residue):
    layout = {k: {"dtype": dt.value, "shape": list(s), "data_offsets": [0, 0]} for k, (dt, s, _) in tensors.items()}
    natural = len(json.dumps(layout, separators=(",", ":")).encode())
    base = natural + 128
    return base + (residue - (8 + base) % 512) % 512


def run_ranks(world, fn):
    res, errs = [None] * world, {}

    def runner(r):
        try:
            res[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    ts = [threading.Thread(target=runner, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    if errs:
        raise errs[min(errs)]
    return res


def corpora() -> None:
    cdir = HERE / "corpora"
    cdir.mkdir(exist_ok=True)
    for old in cdir.glob("*.safetensors"):
        old.unlink()
    rng = np.random.default_rng(0xC0A7)
    cases = []
    matrix = [(b, w, d) for w in (1, 2, 3, 4) for d in (0, 1, 2) for b in ("host", "simdirect")]
    for ci, (backend, world, dim) in enumerate(matrix):
        n_files = int(rng.integers(1, 4))
        files = []
        for f in range(n_files):
            t = random_tensors(rng, int(rng.integers(2, 7)), f"c{ci}f{f}_")
            residue = int(rng.choice([0, 1, 3, 99, 107, 255, 333, 511]))
            name = f"c{ci:02d}_{f}.safetensors"
            (cdir / name).write_bytes(write_file(t, pad_header_to=pad_for_residue(t, residue)))
            files.append(name)
        mapping = {r: [] for r in range(world)}
        for j, f in enumerate(files):
            mapping[j % world].append(str(cdir / f))
        topo = Topology((NumaNode(0, 32, tuple(range(world)), (0,)),))
        cfg = LoaderConfig(backend=backend, topology=topo, auto_release=True)
        group = ProcessGroup(world)
        keys = None

        def rank_main(rank):
            nonlocal keys
            loader = SafeTensorsFileLoader(group, rank=rank, config=cfg)
            loader.add_filenames(mapping)
            fb = loader.copy_files_to_device()
            ks = sorted(fb.keys())
            layout = {Path(p).name: dict(h.dev_offsets) for p, h in fb._hosted.items()}
            got = {}
            for k in ks:
                m = fb.metadata(k)
                if world > 1 and dim < len(m.shape) and m.shape[dim] >= world:
                    v = fb.get_sharded(k, dim)
                    kind = "shard"
                else:
                    v = fb.get_tensor(k)
                    kind = "full"
                got[k] = [kind, list(v.shape), hashlib.sha256(v.tobytes()).hexdigest()]
            fb.close()
            loader.close()
            return got, layout

        results = run_ranks(world, rank_main)
        layouts = {}
        for _, lay in results:
            layouts.update(lay)
        cases.append({"id": ci, "backend": backend, "world": world, "dim": dim, "files": files,
                      "mapping": {str(r): [Path(p).name for p in ps] for r, ps in mapping.items()},
                      "ranks": [g for g, _ in results], "layouts": layouts})
    (cdir / "expect.json").write_text(json.dumps({"generator": "aggload (reference) loader, thread ranks",
                                                  "cases": cases}, indent=1, sort_keys=True))


if __name__ == "__main__":
    os.chdir(HERE)
    conv_vectors()
    corpora()
    print("golden fixtures written to", HERE)
