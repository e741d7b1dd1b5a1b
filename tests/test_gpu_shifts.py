"""Device Ritz values against the reference's splu-based
pencil_ritz_sets (tests/golden/ref_ritz.npz), and the shifts they produce
against the pinned shift files."""

import os

import numpy as np
import pytest

from conftest import GOLD
from paper_2312_02891_b200 import configs as cfgs
from paper_2312_02891_b200 import shifts as S

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _match(got, want, rtol):
    """Every reference Ritz value has a device Ritz value within rtol (relative
    to the set's largest modulus), and the counts agree."""
    assert got.size == want.size, (got.size, want.size)
    scale = np.abs(want).max()
    for w in want:
        assert np.min(np.abs(got - w)) <= rtol * scale, (w, got)


@pytest.mark.parametrize("name", ["c1", "c2", "c3s", "c5s"])
def test_device_ritz_sets_and_shifts_match_reference(name):
    gold = np.load(os.path.join(GOLD, "ref_ritz.npz"))
    A, B, M, C, f, g = cfgs.build_problem(name)
    stats = {}
    rA = S.pencil_ritz_sets(A, M, source="A-side", stats=stats)
    rB = S.pencil_ritz_sets(B, C, source="B-side", stats=stats)
    for side, (d, inv) in (("A", rA), ("B", rB)):
        _match(d.values, gold[f"{name}_{side}_direct"], 1e-9)
        _match(inv.values, gold[f"{name}_{side}_inverse"], 1e-7)
    assert all(v["base_solve_unconverged"] == 0 for v in stats.values())
    seq = S.heuristic_shifts(rA, rB, npairs=cfgs.CONFIGS[name].npairs)
    pinned, _ = cfgs.CONFIGS[name].load_shift_pairs()
    assert len(seq.pairs) == len(pinned)
    for (a, b), (pa, pb) in zip(seq.pairs, pinned):
        assert abs(a - pa) <= 1e-6 * abs(pa) and abs(b - pb) <= 1e-6 * abs(pb)
