"""Shift generation host logic against the reference: the
greedy picker and the objective on the reference's own Ritz sets
(tests/golden/ref_ritz.npz, from shifts.py:101-129 with splu) reproduce the
pinned shift files bit for bit."""

import os

import numpy as np
import pytest

from conftest import GOLD
from paper_2312_02891_b200 import configs as cfgs
from paper_2312_02891_b200 import shifts as S

NAMES = ["c1", "c2", "c3s", "c5s"]


def ritz(gold, name, side):
    src = f"{side}-side"
    return (S.RitzSet(gold[f"{name}_{side}_direct"], src, "direct"),
            S.RitzSet(gold[f"{name}_{side}_inverse"], src, "inverse"))


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "ref_ritz.npz"))


@pytest.mark.parametrize("name", NAMES)
def test_heuristic_shifts_match_pinned_reference_shifts(gold, name):
    seq = S.heuristic_shifts(ritz(gold, name, "A"), ritz(gold, name, "B"),
                             npairs=cfgs.CONFIGS[name].npairs)
    pinned, cyclic = cfgs.CONFIGS[name].load_shift_pairs()
    assert seq.pairs == pinned and seq.cyclic == cyclic


@pytest.mark.parametrize("name", NAMES)
def test_shift_objective_matches_reference(gold, name):
    pinned, _ = cfgs.CONFIGS[name].load_shift_pairs()
    got = S.shift_objective([a for a, _ in pinned], [b for _, b in pinned],
                            ritz(gold, name, "A"), ritz(gold, name, "B"))
    assert got == float(gold[f"{name}_objective"])


def test_shift_objective_edge_cases():
    lam = S.RitzSet(np.array([-1.0, -2.0]), "A-side", "direct")
    mu = S.RitzSet(np.array([-3.0]), "B-side", "direct")
    # a denominator at zero: lambda + beta = 0 -> infinity sentinel (shifts.py:155-156)
    assert S.shift_objective([-3.0], [1.0], lam, mu) == S.INF
    # no pairs: empty product
    assert S.shift_objective([], [], lam, mu) == 1.0
    with pytest.raises(ValueError):
        S.shift_objective([-1.0], [], lam, mu)


def test_heuristic_shifts_rejects_unstable_candidates():
    lam = S.RitzSet(np.array([1.0, 2.0]), "A-side", "direct")
    mu = S.RitzSet(np.array([-1.0]), "B-side", "direct")
    with pytest.raises(ValueError):
        S.heuristic_shifts(lam, mu, npairs=2)


def test_ritzset_rejects_nonfinite():
    with pytest.raises(ValueError):
        S.RitzSet(np.array([np.nan]), "A-side", "direct")
