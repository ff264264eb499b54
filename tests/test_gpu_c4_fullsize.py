"""Parity at the default bench's full size and launch configuration (C4 at N = 1, BASELINE.json
configs[3]): 10M entries built as bench.py builds them, one 16,384-query push batch, 24 sampled
rows against the fp64 oracle over all 10M entries (see tests/fullsize_parity.py)."""
import pytest

from tests.fullsize_parity import run

pytestmark = pytest.mark.gpu


def test_c4_full_size_sampled_parity(oracle_mod):
    rep = run(oracle_mod, "c4", 24)
    print(rep)
    assert rep["samples"] == 24 and rep["exempt"] <= 2 and rep["hits"] > 0
