"""Summarise ncu captures into small JSON files for profiles/ (run here, no GPU).

    python tools/summarize_ncu.py gpurun_out/prof_clone.ncu-rep ... > profiles/rNN_ncu_full.json
    python tools/summarize_ncu.py --launches gpurun_out/ncu_launches.csv > profiles/rNN_ncu_launches.json
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "sm__maximum_warps_per_active_cycle_pct",
    "smsp__inst_executed.sum",
    "lts__t_bytes.sum",
    "l1tex__t_bytes.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "gpc__cycles_elapsed.max",
]


def full(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{vals[i]} {units[i]}".strip()
        try:
            t = float(vals[hdr.index("gpu__time_duration.sum")])
            tu = units[hdr.index("gpu__time_duration.sum")]
            scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(tu, 1e-9)
            rd = float(vals[hdr.index("dram__bytes_read.sum")])
            wr = float(vals[hdr.index("dram__bytes_write.sum")])
            bu = units[hdr.index("dram__bytes_read.sum")]
            bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu, 1)
            d["traffic_bytes"] = (rd + wr) * bscale
            d["dram_GBps"] = (rd + wr) * bscale / (t * scale) / 1e9
        except (ValueError, IndexError):
            pass
        res.append(d)
    return {"report": rep, "launches": res}


def launches(path: str) -> list:
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    out = {}
    for r in rows:
        d = out.setdefault(r["ID"], {"kernel": r["Kernel Name"][:80], "grid": r["Grid Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"])
    return list(out.values())


def launch_shares(path: str) -> dict:
    """Aggregate a launch list per kernel: launches, summed device time and
    DRAM bytes, share of the summed time (ncu serialises launches and runs
    them cold-cache: compare SHARES with the live bench, not absolutes)."""
    rows = launches(path)
    agg: dict[str, dict] = {}
    for r in rows:
        a = agg.setdefault(r["kernel"], {"launches": 0, "time_ns": 0.0, "dram_bytes": 0.0})
        a["launches"] += 1
        a["time_ns"] += r.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
    total = sum(a["time_ns"] for a in agg.values()) or 1.0
    for a in agg.values():
        a["share_of_time"] = round(a["time_ns"] / total, 4)
        a["dram_GBps"] = round(a["dram_bytes"] / a["time_ns"], 1) if a["time_ns"] else None
    top = sorted(rows, key=lambda r: -r.get("gpu__time_duration.sum", 0.0))[:8]
    for r in top:
        t = r.get("gpu__time_duration.sum", 0.0)
        b = r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
        r["dram_GBps"] = round(b / t, 1) if t else None
    return {"source": path, "launches": len(rows), "per_kernel": agg, "longest_launches": top}


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    elif sys.argv[1] == "--shares":
        print(json.dumps(launch_shares(sys.argv[2]), indent=1))
    else:
        print(json.dumps([full(r) for r in sys.argv[1:]], indent=1))
