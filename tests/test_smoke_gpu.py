"""The driver's round-end smoke (``__graft_entry__.smoke()``) as a GPU test:
one odd-header file through the simdirect landing, a bf16->f16 cast, a
realigned f32 column shard and a u8 tensor, checked against the oracle."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


def test_graft_entry_smoke():
    import __graft_entry__

    __graft_entry__.smoke()
