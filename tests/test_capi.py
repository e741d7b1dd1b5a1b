"""The C-ABI library loads and exports exactly what include/sylvadi_b200.h
declares (CPU: no compute calls); host-side helpers of the product path."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2312_02891_b200 import _build, _lib
from paper_2312_02891_b200 import adi as padi
from paper_2312_02891_b200.device import product_norm_from_grams, sigma_max_from_gram
from oracle import sylvadi_oracle as orc

from conftest import REPO

HEADER = os.path.join(REPO, "include", "sylvadi_b200.h")


def header_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sad_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _lib.load()


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_lib.SIGNATURES)


def test_library_exports_every_header_symbol(lib):
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in header_symbols():
        assert hasattr(raw, name), name
    assert lib.sad_version() == 1


def test_status_codes_map_to_reference_exceptions():
    with pytest.raises(ValueError):
        _lib.check(_lib.SAD_EINVAL)
    with pytest.raises(_lib.FactorizationBreakdown):
        _lib.check(_lib.SAD_EBREAKDOWN)
    with pytest.raises(MemoryError):
        _lib.check(_lib.SAD_ENOMEM)
    with pytest.raises(_lib.DeviceError):
        _lib.check(_lib.SAD_ECUDA)


def test_sm100a_cubin_embedded(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


# -- host-side product logic (scalars / Gram algebra) ----------------------------

def test_product_tolerances_match_oracle(rng):
    for strat in ("fixed", "dynamic_mid", "dynamic_mid_bl", "dynamic_b", "dynamic_b_bl",
                  "direct_a_iter_b", "iter_a_direct_b"):
        cfg = padi.AdiConfig(strategy=strat, gap_budget=3e-7, kmax=40)
        ocfg = orc.Config(strategy=strat, gap_budget=3e-7, kmax=40)
        for k in (1, 3, 9):
            uu, vv = 10.0 ** rng.uniform(-12, -9, 2)
            eh = padi.tolerance_budget(cfg, k, uu, vv)
            assert eh == orc.tolerance_budget(ocfg, k, uu, vv)
            nw, nt = 10.0 ** rng.uniform(-8, 0, 2)
            dec = padi.choose_tolerances(cfg, k, nw, nt, eh)
            assert (dec.delta_A, dec.delta_B, dec.clamped_A_min, dec.clamped_B_min) == \
                orc.choose_tolerances(ocfg, k, nw, nt, eh)


def test_product_known_answers():
    cfg = padi.AdiConfig(strategy="dynamic_mid", gap_budget=1e-8, kmax=50)
    assert abs(padi.tolerance_budget(cfg, 1) - 8.5786e-12) < 1e-16
    assert abs(padi.tolB_from_tolA(1e-4, 1e-8, 3.0, 1e-5, 2e-3) - 1.0606e-6) < 1e-9
    cfg = padi.AdiConfig(strategy="fixed", outer_tolerance=1e-8)
    dec = padi.choose_tolerances(cfg, 1, 1.0, 1.0, 1e-12)
    assert dec.delta_A == dec.delta_B == 5e-10
    with pytest.raises(ValueError):
        padi.AdiConfig(outer_tolerance=2.0)
    with pytest.raises(ValueError):
        padi.AdiConfig(delta_min_A=0.2, delta_max_A=0.1)


def test_gram_norms_match_svd_qr(rng):
    for r in (1, 2, 3, 8):
        w = rng.standard_normal((40, r)) + 1j * rng.standard_normal((40, r))
        t = rng.standard_normal((25, r)) + 1j * rng.standard_normal((25, r))
        ref = orc.computed_residual_norm(w, t)
        got = product_norm_from_grams(w.conj().T @ w, t.conj().T @ t)
        assert abs(got - ref) <= 1e-12 * ref
        assert abs(sigma_max_from_gram(w.conj().T @ w) - orc.block_norm(w)) <= 1e-13 * orc.block_norm(w)


def test_shift_sequence_roundtrip(tmp_path):
    from paper_2312_02891_b200 import ShiftSequence
    seq = ShiftSequence(pairs=[(-1 + 2j, -3 + 0j), (-4.5, -0.25 - 1j)], cyclic=True)
    p = str(tmp_path / "s.json")
    seq.to_json(p)
    back = ShiftSequence.from_json(p)
    assert back.pairs == seq.pairs
    assert back.at(3) == seq.at(1)
    with pytest.raises(IndexError):
        ShiftSequence(pairs=[(-1, -1)], cyclic=False).at(2)


def test_report_csv_schema(tmp_path):
    rep = padi.SolveReport()
    rep.records.append(padi.StepRecord(1, 0.5, 1e-9, 2e-9, 3e-10, 4e-10, 5, 6, 1e-9, 2e-9, 1.25))
    p = tmp_path / "r.csv"
    rep.to_csv(str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == padi.CSV_HEADER
    assert lines[1].startswith("1,5.0000000000000000e-01,")
    assert lines[1].endswith(",5,6,1.0000000000000001e-09,2.0000000000000001e-09,1.250")


def test_problem_validation_matches_reference():
    import scipy.sparse as sp
    A = sp.csr_matrix(-np.eye(4))
    B = sp.csr_matrix(-np.eye(3))
    with pytest.raises(ValueError):
        padi.SylvesterProblem(A=A, B=B, f=np.ones((4, 2)), g=np.ones((3, 2)))
    prob = padi.SylvesterProblem(A=A, B=B, f=np.ones(4), g=np.ones(3))
    assert prob.f.shape == (4, 1) and prob.r == 1
