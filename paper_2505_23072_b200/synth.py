"""Synthetic checkpoints of the benchmark architectures (no network, no real
weights): HF tensor names/shapes/order, HF-style file splits, values fp32
N(0, 0.02) rounded to the file dtype (RNE) from per-tensor seeded generators.

Architectures (BASELINE.json configs):
  gpt2        GPT-2 small fp32, 148 tensors, 1 file, 497,759,232 B
  llama2-7b   bf16, 291 tensors, 2 files, 13,476,831,232 B
  llama2-13b  bf16, 363 tensors, 3 files, 26,031,728,640 B
  llama2-70b  bf16, 723 tensors, 15 files, 137,953,296,384 B (GQA, 8 KV heads)
  bloom-176b  bf16, 845 tensors, 72 files, 352,494,542,848 B

``shard_dim`` gives the Megatron tensor-parallel split used by the benchmarks
(PAPER.md:159-161): column-parallel weights on dim 0, row-parallel on dim 1,
norms and row-parallel biases replicated (``None`` -> get_tensor).

Reference counterpart: the seeded corpus generator of cli.py:85-122 and the
fixture writer format.py:295-338 (re-implemented here as a streaming writer).
"""

from __future__ import annotations

import math
import os
from pathlib import Path

import numpy as np

from .format import DType, write_file_stream

Entry = tuple[str, DType, tuple[int, ...]]


def _gpt2() -> list[Entry]:
    H, V, P, L = 768, 50257, 1024, 12
    f = DType.F32
    out: list[Entry] = [("wte.weight", f, (V, H)), ("wpe.weight", f, (P, H))]
    for i in range(L):
        p = f"h.{i}."
        out += [(p + "ln_1.weight", f, (H,)), (p + "ln_1.bias", f, (H,)),
                (p + "attn.c_attn.weight", f, (H, 3 * H)), (p + "attn.c_attn.bias", f, (3 * H,)),
                (p + "attn.c_proj.weight", f, (H, H)), (p + "attn.c_proj.bias", f, (H,)),
                (p + "ln_2.weight", f, (H,)), (p + "ln_2.bias", f, (H,)),
                (p + "mlp.c_fc.weight", f, (H, 4 * H)), (p + "mlp.c_fc.bias", f, (4 * H,)),
                (p + "mlp.c_proj.weight", f, (4 * H, H)), (p + "mlp.c_proj.bias", f, (H,))]
    out += [("ln_f.weight", f, (H,)), ("ln_f.bias", f, (H,))]
    return out


def _llama(H: int, I: int, L: int, kv: int, V: int = 32000) -> list[Entry]:
    b = DType.BF16
    out: list[Entry] = [("model.embed_tokens.weight", b, (V, H))]
    for i in range(L):
        p = f"model.layers.{i}."
        out += [(p + "input_layernorm.weight", b, (H,)),
                (p + "self_attn.q_proj.weight", b, (H, H)),
                (p + "self_attn.k_proj.weight", b, (kv, H)),
                (p + "self_attn.v_proj.weight", b, (kv, H)),
                (p + "self_attn.o_proj.weight", b, (H, H)),
                (p + "post_attention_layernorm.weight", b, (H,)),
                (p + "mlp.gate_proj.weight", b, (I, H)),
                (p + "mlp.up_proj.weight", b, (I, H)),
                (p + "mlp.down_proj.weight", b, (H, I))]
    out += [("model.norm.weight", b, (H,)), ("lm_head.weight", b, (V, H))]
    return out


def _bloom() -> list[Entry]:
    H, V, L = 14336, 250880, 70
    b = DType.BF16
    out: list[Entry] = [("word_embeddings.weight", b, (V, H)),
                        ("word_embeddings_layernorm.weight", b, (H,)),
                        ("word_embeddings_layernorm.bias", b, (H,))]
    for i in range(L):
        p = f"h.{i}."
        out += [(p + "input_layernorm.weight", b, (H,)), (p + "input_layernorm.bias", b, (H,)),
                (p + "self_attention.query_key_value.weight", b, (3 * H, H)),
                (p + "self_attention.query_key_value.bias", b, (3 * H,)),
                (p + "self_attention.dense.weight", b, (H, H)),
                (p + "self_attention.dense.bias", b, (H,)),
                (p + "post_attention_layernorm.weight", b, (H,)),
                (p + "post_attention_layernorm.bias", b, (H,)),
                (p + "mlp.dense_h_to_4h.weight", b, (4 * H, H)),
                (p + "mlp.dense_h_to_4h.bias", b, (4 * H,)),
                (p + "mlp.dense_4h_to_h.weight", b, (H, 4 * H)),
                (p + "mlp.dense_4h_to_h.bias", b, (H,))]
    out += [("ln_f.weight", b, (H,)), ("ln_f.bias", b, (H,))]
    return out


ARCHS = {
    "gpt2": (_gpt2, None),
    "llama2-7b": (lambda: _llama(4096, 11008, 32, 4096), 10_000_000_000),
    "llama2-13b": (lambda: _llama(5120, 13824, 40, 5120), 10_000_000_000),
    "llama2-70b": (lambda: _llama(8192, 28672, 80, 1024), 9_900_000_000),
    "bloom-176b": (_bloom, "per-layer"),
}


def entries(arch: str, layers: int | None = None) -> list[Entry]:
    """All tensors, or a prefix of the transformer blocks (embeddings and the
    final norm / lm_head kept) when ``layers`` is given — the same shapes at a
    size one GPU and the box's disk can hold for parity tests."""
    ents = ARCHS[arch][0]()
    if layers is None:
        return ents

    def block(name: str) -> int | None:
        parts = name.split(".")
        for i, p in enumerate(parts[:-1]):
            if p in ("layers", "h") and parts[i + 1].isdigit():
                return int(parts[i + 1])
        return None

    return [e for e in ents if (block(e[0]) is None or block(e[0]) < layers)]


def nbytes(e: Entry) -> int:
    return math.prod(e[2]) * e[1].size_bytes


def split_files(arch: str, ents: list[Entry] | None = None, max_bytes: int | None = None) -> list[list[Entry]]:
    """HF-style split: greedy fill up to the max shard size (Llama), one file
    per transformer block (Bloom: embeddings / 70 layers / ln_f), or one file."""
    ents = ents if ents is not None else entries(arch)
    rule = ARCHS[arch][1] if max_bytes is None else max_bytes
    if rule is None:
        return [ents]
    if rule == "per-layer":
        groups: dict[str, list[Entry]] = {}
        for e in ents:
            key = e[0].split(".")[1] if e[0].startswith("h.") else ("embed" if "word_emb" in e[0] else "final")
            groups.setdefault(key, []).append(e)
        return list(groups.values())
    files, cur, size = [], [], 0
    for e in ents:
        if cur and size + nbytes(e) > rule:
            files.append(cur)
            cur, size = [], 0
        cur.append(e)
        size += nbytes(e)
    if cur:
        files.append(cur)
    return files


_COL = ("q_proj", "k_proj", "v_proj", "gate_proj", "up_proj", "embed_tokens", "lm_head",
        "query_key_value", "dense_h_to_4h", "word_embeddings.weight")
_ROW = ("o_proj", "down_proj", "self_attention.dense.weight", "dense_4h_to_h.weight")


def shard_dim(name: str, shape: tuple[int, ...]) -> int | None:
    """Megatron split for the Llama/Bloom benchmarks; None = replicate."""
    if any(k in name for k in _ROW):
        return 1
    if any(k in name for k in _COL):
        return 0
    return None


# ------------------------------------------------------------------------ values
def _bf16_rne(x: np.ndarray) -> np.ndarray:
    u = x.view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def host_values(e: Entry, seed: int) -> np.ndarray:
    """CPU generation (small corpora): N(0, 0.02) fp32 -> dtype, RNE."""
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(math.prod(e[2]), dtype=np.float32) * np.float32(0.02))
    if e[1] is DType.F32:
        return x
    if e[1] is DType.BF16:
        return _bf16_rne(x)
    if e[1] is DType.F16:
        return x.astype(np.float16)
    raise ValueError(f"no value generator for {e[1]}")


def device_values(e: Entry, seed: int, device: str = "cuda") -> np.ndarray:
    """GPU generation for the multi-GB corpora; returns host bytes (numpy)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    t = torch.randn(math.prod(e[2]), generator=g, device=device, dtype=torch.float32) * 0.02
    tdt = {DType.F32: torch.float32, DType.BF16: torch.bfloat16, DType.F16: torch.float16}[e[1]]
    t = t.to(tdt)
    return t.view(torch.uint8).cpu().numpy()


def body_pad(ents: list[Entry], header: str) -> int | None:
    """pad_header_to for the header mode: 'aligned' (body % 8 == 0, as real
    writers), 'odd' (aligned + 1: every tensor lands misaligned on the
    GDS-shaped backends), or 'natural' (compact JSON, whatever it gives)."""
    if header == "natural":
        return None
    import json

    layout, cur = {}, 0
    for name, dt, shape in ents:
        nb = math.prod(shape) * dt.size_bytes
        layout[name] = {"dtype": dt.value, "shape": list(shape), "data_offsets": [cur, cur + nb]}
        cur += nb
    n = len(json.dumps(layout, separators=(",", ":")).encode())
    aligned = n + (-(8 + n)) % 8
    return aligned + (1 if header == "odd" else 0)


def generate(arch: str, outdir: str | os.PathLike, header: str = "aligned", seed: int = 0,
             device: str | None = None, files: list[int] | None = None, layers: int | None = None,
             max_bytes: int | None = None) -> list[Path]:
    """Write the checkpoint; returns the file paths (all of them, even when
    ``files`` restricts which ones are (re)written). ``layers`` keeps only the
    first transformer blocks; ``max_bytes`` overrides the file split size."""
    outdir = Path(outdir)
    outdir.mkdir(parents=True, exist_ok=True)
    groups = split_files(arch, entries(arch, layers), max_bytes)
    paths = []
    base = 0
    for fi, ents in enumerate(groups):
        p = outdir / f"model-{fi + 1:05d}-of-{len(groups):05d}.safetensors"
        paths.append(p)
        if files is None or fi in files:
            def produce(i, ents=ents, base=base):
                e = ents[i]
                if device:
                    return device_values(e, seed * 1_000_003 + base + i, device)
                return host_values(e, seed * 1_000_003 + base + i)
            write_file_stream(p, ents, produce, pad_header_to=body_pad(ents, header))
        base += len(ents)
    return paths


def total_bytes(arch: str) -> int:
    return sum(nbytes(e) for e in entries(arch))
