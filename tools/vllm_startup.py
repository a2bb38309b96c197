"""vLLM model-load time on one B200 with three weight loaders (the paper's
application benchmark): safetensors (vLLM default),
upstream fastsafetensors 0.3.1 (``load_format="fastsafetensors"``), and this
loader behind the same load format (paper_2505_23072_b200.vllm_loader).

    python tools/vllm_startup.py [--arch llama2-7b] [--runs 2]

Each run is a fresh process (engine in-process, eager mode, no tokenizer);
the synthetic checkpoint (random weights, HF names) is page-cache warm.
Prints one JSON line per run with vLLM's own "Loading weights took" time and
the wall time of LLM(...) construction.
"""

from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "llama2-7b": dict(hidden_size=4096, intermediate_size=11008, num_hidden_layers=32, num_attention_heads=32,
                      num_key_value_heads=32),
    "llama2-13b": dict(hidden_size=5120, intermediate_size=13824, num_hidden_layers=40, num_attention_heads=40,
                       num_key_value_heads=40),
}

CHILD = r"""
import os, sys, time, json
sys.path.insert(0, {root!r})
mode = {mode!r}
if mode == "ours":
    from paper_2505_23072_b200 import vllm_loader
    vllm_loader.install()
if mode == "fastsafetensors":
    # vLLM asks upstream for GDS at TP=1 (nogds=False); without nvidia-fs cuFile's
    # compat-mode driver open hangs on this box, so force its no-GDS path
    from vllm.model_executor.model_loader import weight_utils as wu
    _orig = wu._init_fastsafetensors_loader
    wu._init_fastsafetensors_loader = lambda pg, device, f_list, nogds=False: _orig(pg, device, f_list, nogds=True)
from vllm import LLM
t0 = time.perf_counter()
llm = LLM(model={model!r}, load_format=("safetensors" if mode == "safetensors" else "fastsafetensors"),
          skip_tokenizer_init=True, enforce_eager=True, gpu_memory_utilization=0.6, max_model_len=256,
          dtype="bfloat16", compilation_config=0)
print("LLM_READY_S", time.perf_counter() - t0, flush=True)
"""


def make_model(arch: str, root: Path) -> Path:
    from bench import ensure_data

    paths = ensure_data(arch, str(root / "data"), "aligned", 0, 1, None)
    d = root / arch
    d.mkdir(parents=True, exist_ok=True)
    for p in paths:
        link = d / p.name
        if not link.exists():
            link.symlink_to(p)
    cfg = {"architectures": ["LlamaForCausalLM"], "model_type": "llama", "vocab_size": 32000,
           "max_position_embeddings": 4096, "rms_norm_eps": 1e-5, "hidden_act": "silu", "torch_dtype": "bfloat16",
           "tie_word_embeddings": False, "bos_token_id": 1, "eos_token_id": 2, **CONFIGS[arch]}
    (d / "config.json").write_text(json.dumps(cfg))
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", default="llama2-7b")
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--modes", default="safetensors,fastsafetensors,ours")
    ap.add_argument("--root", default="/tmp/hl_vllm")
    ap.add_argument("--timeout", type=int, default=420)
    args = ap.parse_args()
    model = make_model(args.arch, Path(args.root))
    from bench import warm_cache

    files = sorted(model.glob("*.safetensors"))
    total = sum(os.path.getsize(p) for p in files)
    env = dict(os.environ, VLLM_ENABLE_V1_MULTIPROCESSING="0", HF_HUB_OFFLINE="1", TRANSFORMERS_OFFLINE="1")
    for run in range(args.runs):
        for mode in args.modes.split(","):
            warm_cache([p.resolve() for p in files])
            t0 = time.perf_counter()
            try:
                r = subprocess.run([sys.executable, "-c", CHILD.format(root=str(ROOT), mode=mode, model=str(model))],
                                   capture_output=True, text=True, env=env, timeout=args.timeout)
                rc, log = r.returncode, r.stdout + r.stderr
            except subprocess.TimeoutExpired as e:
                rc = "timeout"
                log = (e.stdout or b"").decode(errors="replace") + (e.stderr or b"").decode(errors="replace")
            wall = time.perf_counter() - t0
            m = re.search(r"Loading weights took ([0-9.]+) seconds", log)
            ml = re.search(r"Model loading took ([0-9.]+) GiB(?: memory)? and ([0-9.]+) seconds", log)
            ready = re.search(r"LLM_READY_S ([0-9.]+)", log)
            line = {"mode": mode, "run": run, "rc": rc, "arch": args.arch, "bytes": total,
                    "load_weights_s": float(m.group(1)) if m else None,
                    "model_loading_s": float(ml.group(2)) if ml else None,
                    "llm_ready_s": float(ready.group(1)) if ready else None, "process_wall_s": round(wall, 2)}
            if m:
                line["load_weights_GBps"] = round(total / float(m.group(1)) / 1e9, 2)
            if rc != 0:
                line["tail"] = log[-1500:]
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
