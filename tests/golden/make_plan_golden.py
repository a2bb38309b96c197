"""Golden transfer plans from the REFERENCE's build_plan (transfer.py:211-302)
over random file sets x backends x block sizes x topologies (build container
only). Re-run:  python tests/golden/make_plan_golden.py  -> plan_cases.json
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

from aggload.transfer import FileSpec, NumaNode, Topology, build_plan  # noqa: E402  (reference, read-only)


def main():
    rng = np.random.default_rng(11)
    cases = []
    for _ in range(150):
        nodes = int(rng.integers(1, 3))
        cpus = int(rng.integers(1, 48))
        topo = {"nodes": [{"node_id": i, "physical_cpus": cpus, "device_ids": [i], "storage_ids": [i]}
                          for i in range(nodes)]}
        files = [{"file_id": f"f{i}", "size": int(rng.integers(0, 50000)), "storage_id": int(rng.integers(0, 3)),
                  "body_offset": int(rng.integers(8, 900))} for i in range(int(rng.integers(1, 7)))]
        files = [f for f in files if f["size"] >= f["body_offset"]] or [{"file_id": "f", "size": 1000,
                                                                          "storage_id": 0, "body_offset": 8}]
        backend = ["host", "simdirect"][int(rng.integers(0, 2))]
        block = int(rng.integers(1, 9000))
        devices = [int(d) for d in rng.integers(0, 2, size=int(rng.integers(1, 3)))]
        cap = int(rng.integers(1, 20))
        mins = {f["file_id"]: int(rng.integers(0, 60000)) for f in files if rng.random() < 0.3}
        t = Topology(tuple(NumaNode(n["node_id"], n["physical_cpus"], tuple(n["device_ids"]), tuple(n["storage_ids"]))
                           for n in topo["nodes"]))
        plan = build_plan([FileSpec(**f) for f in files], backend, block_size=block, topology=t,
                          target_devices=devices, worker_cap=cap, min_buffer_bytes=mins)
        cases.append({"topology": topo, "files": files, "backend": backend, "block": block, "devices": devices,
                      "cap": cap, "min_buffer_bytes": mins,
                      "expect": {"workers": plan.workers, "cross": plan.cross_numa_blocks,
                                 "affinity": [list(a) for a in plan.affinity],
                                 "blocks": [[b.file_id, b.file_off, b.len, b.buffer_id, b.dev_off, b.worker_id]
                                            for b in plan.blocks],
                                 "buffers": [[b.buffer_id, b.file_id, b.size, b.device_id, b.storage_node]
                                             for b in plan.buffers]}})
    (HERE / "plan_cases.json").write_text(json.dumps({"cases": cases}) + "\n")
    print(f"wrote {len(cases)} plans")


if __name__ == "__main__":
    main()
