"""hl_gather alone on Llama-2-7B-shaped descriptor batches (no files).

Variants (one launch = all 291 tensors of the checkpoint unless noted):
  clone      aligned bf16 copy (get_tensors / auto-release clones)
  realign    every source misaligned by 1 byte (odd header on the GDS landing)
  cast       bf16 -> f16 (C5's on-device cast), aligned source
  castodd    bf16 -> f16 from a misaligned source
  f32f16     f32 -> f16 (GPT-2 fp32 checkpoint cast)
  pack8      owner-side TP=8 pack of every sharded weight (dim 0 / dim 1 Megatron splits)
  pack8cast  the same with the bf16 -> f16 cast fused (C5's owner pack)
  cols8      only the dim-1 (column) shards of pack8: the 2-D TMA tile kernel
  cols8cast  the same with the cast (tile_cast_kernel)

Prints one JSON line per variant: algorithmic GB/s (read+write) from CUDA
events around each launch, and the fraction of MEASURED_PEAKS.json hbm_gbs.
This script is also the ncu target (tools/profile.sh).
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2505_23072_b200 import _native, kernels, synth  # noqa: E402
from paper_2505_23072_b200.format import DType  # noqa: E402


def batches(variant: str, src: torch.Tensor, dst: torch.Tensor, ents):
    base_s, base_d = src.data_ptr(), dst.data_ptr()
    descs, so, do = [], 0, 0
    shift = 1 if variant in ("realign", "castodd", "f32f16odd", "f16f32odd") else 0
    for name, dt, shape in ents:
        n = math.prod(shape)
        if variant in ("f32f16", "f32f16odd"):
            sdt, ddt = DType.F32, DType.F16
        elif variant in ("f16f32", "f16f32odd"):
            sdt, ddt = DType.F16, DType.F32
        elif variant == "bf16f32":
            sdt, ddt = DType.BF16, DType.F32
        elif variant in ("cast", "castodd", "pack8cast", "cols8cast"):
            sdt, ddt = DType.BF16, DType.F16
        else:
            sdt, ddt = DType.BF16, DType.BF16
        if variant.startswith(("pack8", "cols8")):
            d = synth.shard_dim(name, shape)
            if d is None or (variant.startswith("cols8") and d == 0):
                continue
            for r in range(8):
                lo, hi = kernels.shard_bounds(shape[d], 8, r)
                descs.append(kernels.shard_desc(base_s + so, shape, d, lo, hi, base_d + do, sdt, ddt))
                do += -(-(n // shape[d] * (hi - lo) * ddt.size_bytes) // 256) * 256
        else:
            descs.append(kernels.copy_desc(base_s + so + shift, base_d + do, n, sdt, ddt))
            do += -(-(n * ddt.size_bytes) // 256) * 256
        so += -(-(n * sdt.size_bytes) // 256) * 256
    return descs, so + 64, do + 64


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="clone,realign,cast,castodd,f32f16,f32f16odd,f16f32,f16f32odd,bf16f32,pack8")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--arch", default="llama2-7b")
    ap.add_argument("--layers", type=int, default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6650.0) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    ents = synth.entries(args.arch, args.layers)
    for variant in args.variants.split(","):
        if variant in ("f32f16", "f32f16odd"):
            ents_v = [(n, DType.F32, s) for n, _, s in ents]
        else:
            ents_v = ents
        # buffer sizes from a dry run (null bases, never launched)
        _, ssz, dsz = batches(variant, torch.empty(0, device=dev), torch.empty(0, device=dev), ents_v)
        src = torch.empty(ssz, dtype=torch.uint8, device=dev)
        src.view(-1)[: ssz // 2 * 2].view(torch.int16).random_(-16000, 16000)
        dst = torch.empty(dsz, dtype=torch.uint8, device=dev)
        descs, _, _ = batches(variant, src, dst, ents_v)
        nbytes = kernels.algorithmic_bytes(descs)
        times = []
        kernels.TIMING = []
        _native.gather_timing(True)
        for i in range(args.iters + 2):
            kernels.run(descs, dev)
            torch.cuda.synchronize()
            timed = kernels.timings()
            if i >= 2:
                times.append(sum(t for t, _ in timed))
                nl = len(timed)
        _native.gather_timing(False)
        kernels.TIMING = None
        ms = sorted(times)[len(times) // 2]
        gbs = nbytes / (ms / 1e3) / 1e9
        print(json.dumps({"variant": variant, "descriptors": len(descs), "algorithmic_bytes": nbytes,
                          "ms": round(ms, 4), "GBps": round(gbs, 1), "frac_of_hbm_peak": round(gbs / peak, 4),
                          "kernels_run_calls": nl, "arch": args.arch,
                          "layers": args.layers}), flush=True)
        del src, dst
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
