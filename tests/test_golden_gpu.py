"""The B200 loader against the REFERENCE loader's own outputs.

tests/golden/corpora/expect.json was produced by running the reference
(aggload) loader with thread ranks over these corpora (make_golden.py): per
(backend, world, dim) and per rank, every key's kind/shape/sha256. Here the
same mapping and the same call sequence run through our loader (thread ranks
on one GPU, data moved by hl_gather kernels) and must give identical bytes.
"""

from __future__ import annotations

import hashlib

import pytest

pytest.importorskip("torch")

from conftest import GOLDEN, run_ranks  # noqa: E402
from paper_2505_23072_b200 import LoaderConfig, ProcessGroup, SafeTensorsFileLoader  # noqa: E402

pytestmark = pytest.mark.gpu

CORPORA = GOLDEN / "corpora"


def _run_case(case, backend=None, auto_release=True):
    world, dim = case["world"], case["dim"]
    mapping = {int(r): [str(CORPORA / f) for f in fs] for r, fs in case["mapping"].items()}
    group = ProcessGroup(world)
    cfg = LoaderConfig(backend=backend or case["backend"], auto_release=auto_release)

    def rank_main(rank):
        loader = SafeTensorsFileLoader(group, rank=rank, config=cfg)
        loader.add_filenames(mapping)
        fb = loader.copy_files_to_device()
        layout = {p.split("/")[-1]: dict(h.dev_offsets) for p, h in fb._hosted.items()}
        got = {}
        for k in sorted(fb.keys()):
            m = fb.metadata(k)
            if world > 1 and dim < len(m.shape) and m.shape[dim] >= world:
                v, kind = fb.get_sharded(k, dim), "shard"
            else:
                v, kind = fb.get_tensor(k), "full"
            got[k] = [kind, list(v.shape), hashlib.sha256(v.tobytes()).hexdigest()]
        fb.close()
        loader.close()
        return got, layout

    return run_ranks(world, rank_main)


def test_all_golden_cases_bit_exact(golden_cases):
    for case in golden_cases:
        results = _run_case(case)
        for rank, (got, layout) in enumerate(results):
            assert got == case["ranks"][rank], (case["id"], rank)
            if case["backend"] == "simdirect":
                for f, offs in layout.items():
                    assert offs == case["layouts"][f], (case["id"], f)


@pytest.mark.parametrize("backend", ["host", "simdirect", "gds"])
def test_golden_cases_other_backends_and_views(golden_cases, backend):
    """Bytes do not depend on the backend (landing rule) or on auto_release."""
    for case in golden_cases[::5]:
        for auto in (True, False):
            results = _run_case(case, backend=backend, auto_release=auto)
            for rank, (got, _) in enumerate(results):
                assert got == case["ranks"][rank], (case["id"], rank, backend, auto)
