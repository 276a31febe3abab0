"""The verify tool's own pins (SPEC S:455-457 fault injection):
a correct graph passes; one dropped edge is reported as exactly 1 missing,
an injected distance-2 pair as exactly 1 extra, two swapped cells as an
order failure.  CPU only (the oracle's own output is the 'result')."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import oracle  # noqa: E402
import synth  # noqa: E402
from verify import compare, inject, verify  # noqa: E402


@pytest.fixture(scope="module")
def case():
    x = synth.config("C1")["bytes"]
    rc, oc, oe = oracle.build(x)
    assert rc == 0
    return x, oc, oe


def test_correct_graph_passes(case):
    x, oc, oe = case
    rep = verify(x, oc, oe)
    assert rep["ok"] and rep["n_missing"] == 0 and rep["n_extra"] == 0


def test_dropped_edge_is_one_missing(case):
    x, oc, oe = case
    c, e = inject(oc, oe, "drop", seed=3)
    rep = compare(c, e, oc, oe)
    assert not rep["ok"] and rep["n_missing"] == 1 and rep["n_extra"] == 0


def test_distance_two_pair_is_one_extra():
    # (C1's cells are pairwise >= 3 apart except the planted pairs: use a
    # hypercube, where distance-2 pairs abound)
    x = synth.hypercube(6)
    rc, oc, oe = oracle.build(x)
    c, e = inject(oc, oe, "extra")
    rep = compare(c, e, oc, oe)
    assert not rep["ok"] and rep["n_extra"] == 1 and rep["n_missing"] == 0
    i, j = rep["extra"][0]
    assert sum(bin(int(a) ^ int(b)).count("1") for a, b in zip(oc[i], oc[j])) == 2


def test_swapped_cells_fail_the_order(case):
    x, oc, oe = case
    c, e = inject(oc, oe, "swap", seed=5)
    rep = compare(c, e, oc, oe)
    assert not rep["ok"] and not rep["cells_order_ok"] and not rep["cells_ok"]


def test_hypercube_and_arrangement_pass():
    for x in (synth.hypercube(8), synth.config("C3F")["bytes"][:20000]):
        rc, oc, oe = oracle.build(x)
        assert verify(x, oc, oe)["ok"]
