"""Golden outputs of the reference CLI's producer-side tools, made with the
REFERENCE itself (build container only; /root/reference does not exist on the
GPU box). Re-run:  python tests/golden/make_cli_golden.py

For each argument set: `aggload gen` (ref cli.py:81-116) file digests, and
the `inspect` / `shard-plan` JSON documents (ref cli.py:122-164) of the first
file. Written to tests/golden/cli_gen.json; tests/test_cli.py checks that
paper_2505_23072_b200.cli produces identical bytes and documents.
"""

from __future__ import annotations

import contextlib
import hashlib
import io
import json
import sys
import tempfile
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

from aggload.cli import main as ref_main  # noqa: E402  (reference code, read-only import)

CASES = [
    ["--files", "2", "--bytes-per-file", "4096", "--seed", "42", "--dtype", "mixed"],
    ["--files", "3", "--bytes-per-file", "65536", "--seed", "3", "--dtype", "mixed"],
    ["--files", "2", "--bytes-per-file", "64k", "--seed", "7"],
    ["--files", "2", "--bytes-per-file", "1024", "--pad-header", "299"],
    ["--files", "1", "--bytes-per-file", "512", "--pad-header", "99", "--dtype", "BF16"],
    ["--files", "4", "--bytes-per-file", "10007", "--seed", "11", "--dtype", "F64"],
    ["--files", "2", "--bytes-per-file", "3", "--seed", "5", "--dtype", "I64"],
]
PLANS = [("2", "0"), ("2", "1"), ("3", "0"), ("8", "1")]


def run(argv) -> tuple[int, str]:
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = ref_main(argv)
    return rc, buf.getvalue()


def main() -> None:
    out = []
    for args in CASES:
        with tempfile.TemporaryDirectory() as d:
            rc, _ = run(["gen", *args, "--out", d])
            assert rc == 0
            files = sorted(Path(d).glob("*.safetensors"))
            first = str(files[0])
            rc, insp = run(["inspect", first])
            plans = {}
            for w, dim in PLANS:
                rc, doc = run(["shard-plan", first, "--world-size", w, "--dim", dim])
                j = json.loads(doc)
                j.pop("file")
                plans[f"w{w}d{dim}"] = j
            out.append({"args": args, "files": [f.name for f in files],
                        "sha256": [hashlib.sha256(f.read_bytes()).hexdigest() for f in files],
                        "inspect": json.loads(insp), "shard_plan": plans})
    (HERE / "cli_gen.json").write_text(json.dumps({"cases": out}, indent=1) + "\n")
    print(f"wrote {len(out)} cases to {HERE / 'cli_gen.json'}")


if __name__ == "__main__":
    main()
