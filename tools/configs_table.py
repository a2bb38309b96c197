"""Markdown rows of DESIGN.md §5's configs table from bench lines
(profiles/<dir>/*.json, one bench.py JSON line per BASELINE config)."""
import json
import sys
from pathlib import Path

ORDER = ["c1", "c1_f16", "c1_odd_gds", "c2", "c3", "c3_tp2", "c3_tp4", "c4_l24", "c4_l4_tp8", "c5_l8_f16",
         "c5_l2_tp8_f16"]


def row(name, d):
    c, e, io, r = d["config"], d.get("e2e") or {}, d.get("io_roofline") or {}, d.get("roofline") or {}
    cold, cpu = d.get("e2e_cold") or {}, d.get("cpu_baseline") or {}
    planes = d.get("planes")
    if planes:
        val = " / ".join(f"{planes[p]['value']:.1f}" for p in ("ipc", "nccl") if p in planes) + " GB/s (ipc / nccl)"
    else:
        val = f"{d['value']:.1f} GB/s ({d['ms_per_step'] / 1e3:.3f} s)"
    frac = f"{io['e2e_frac_of_h2d']:.2f}" if io.get("e2e_frac_of_h2d") else ""
    cs = f"{cold['value']:.2f}" + (f" ({cold['frac_of_storage']:.2f})" if cold.get("frac_of_storage") else "") \
        if cold else ""
    kern = ""
    if r.get("frac") and not planes:
        k = r.get("kernel", "").replace("hl_gather ", "").split(" (")[0]
        kern = f"{k} {r['frac']:.2f}"
    ref = f"{cpu['value']:.2f} / {cpu['cold']['value']:.2f}" if cpu.get("cold") else ""
    return (f"| {name} | {c['workload']} | {c['tensor_bytes'] / 1e9:.2f} GB | {val} | {frac} | {cs} | {kern} "
            f"| {ref} |")


d = Path(sys.argv[1])
print("| config | workload | tensor bytes | value (warm e2e) | of H2D | cold e2e GB/s (of storage) "
      "| roofline-leg kernel (of HBM peak) | reference warm / cold GB/s |")
print("|---|---|---|---|---|---|---|---|")
for n in ORDER:
    f = d / f"{n}.json"
    if f.exists():
        try:
            print(row(n, json.loads(f.read_text())))
        except (ValueError, KeyError) as e:
            print(f"| {n} | (no line: {type(e).__name__}) |")
