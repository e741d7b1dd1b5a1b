"""GPU verification diagnostics against the oracle and the
reference's own true_residual_norm values."""

import os

import numpy as np
import pytest

from conftest import GOLD
from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200 import configs as cfgs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("K", [1, 37, 300])
@pytest.mark.parametrize("nvec", [1, 2])
def test_tall_skinny_products(rng, cplx, K, nvec):
    from paper_2312_02891_b200 import _lib
    from paper_2312_02891_b200.verify import _Factor
    n = 5003
    X = rng.standard_normal((n, K))
    if cplx:
        X = X + 1j * rng.standard_normal((n, K))
    V = rng.standard_normal((n, nvec)) + 1j * rng.standard_normal((n, nvec))
    F = _Factor(X, n, 0)
    ctx = _lib.context(0)
    s = torch.cuda.current_stream().cuda_stream
    Vd = torch.from_numpy(V).cuda()
    got = F.hgemv(ctx, Vd, s)
    want = X.conj().T @ V
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want)) * np.sqrt(n)
    Cc = rng.standard_normal((K, nvec)) + 1j * rng.standard_normal((K, nvec))
    Y = torch.zeros((n, nvec), dtype=torch.complex128, device="cuda")
    F.gemv(ctx, Cc, Y, s)
    F.gemv(ctx, Cc, Y, s, accumulate=True)
    want = 2.0 * (X @ Cc)
    got = Y.cpu().numpy()
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want)) * np.sqrt(K)


@pytest.mark.parametrize("name", ["c1", "c3s"])
def test_true_residual_norm_matches_reference(name):
    """Device power iteration = the reference's value on its own factors."""
    import paper_2312_02891_b200 as pb
    from paper_2312_02891_b200.verify import true_residual_norm
    gold = np.load(os.path.join(GOLD, f"ref_verify_{name}.npz"))
    A, B, M, C, f, g = cfgs.build_problem(name)
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
    r = f.shape[1]
    gd = gold["gdiag"]
    sol = pb.LowRankSolution(Z=gold["Z"], gammas=gd[::r], Y=gold["Y"], r=r)
    got = true_residual_norm(prob, sol)
    want = float(gold["true_residual_norm"])
    assert abs(got - want) <= 1e-8 * want, (got, want)


def test_true_residual_of_converged_device_run():
    """A converged device ADI run (config 1): the device true residual equals
    the oracle's on the downloaded factors, and the equation is solved to the
    outer tolerance (true residual <= 2 tau ||f g^*||)."""
    import paper_2312_02891_b200 as pb
    from paper_2312_02891_b200.verify import true_residual_norm
    spec = cfgs.CONFIGS["c1"]
    A, B, M, C, f, g = cfgs.build_problem("c1")
    pairs, cyclic = spec.load_shift_pairs()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
    cfg = pb.AdiConfig(strategy=spec.strategy, kmax=spec.kmax, precond_kind_A="jacobi",
                       precond_kind_B="jacobi")
    sol, rep = pb.run(prob, cfg, pb.ShiftSequence(pairs=pairs, cyclic=cyclic),
                      restart=spec.restart, flexible=spec.flexible)
    assert rep.converged
    dev = true_residual_norm(prob, sol)
    host = orc.true_residual_norm(A, B, f, g, sol.Z, sol.Y, sol.gamma_diag())
    assert abs(dev - host) <= 1e-6 * host, (dev, host)
    fg = np.linalg.norm(f) * np.linalg.norm(g)   # = ||f g^*||_2 for r = 1
    assert dev <= 2.0 * cfg.outer_tolerance * fg, dev / fg


def _golden_state(gold, r):
    import paper_2312_02891_b200 as pb
    k = int(gold["steps"])
    SA, SB = gold["S_A"], gold["S_B"]
    return pb.AdiState(k, gold["Z"], gold["Y"], list(gold["gammas"]), gold["w"], gold["t"],
                       float(gold["u"]), float(gold["v"]),
                       [tuple(p) for p in gold["shift_history"]],
                       [SA[:, j * r:(j + 1) * r] for j in range(k)],
                       [SB[:, j * r:(j + 1) * r] for j in range(k)], True)


@pytest.mark.parametrize("name", ["c1", "c3s"])
def test_gap_and_factor_identity_match_reference(name):
    """Device residual_gap / verify_factor_identity (adi.py:632-679) on the
    state the reference's driver retained: the gap equals the reference's
    value, the identity holds to rounding as in the reference, and a defect
    the identity does not absorb (S^A dropped) equals the oracle's value."""
    import paper_2312_02891_b200 as pb
    from paper_2312_02891_b200.verify import residual_gap, verify_factor_identity
    gold = np.load(os.path.join(GOLD, f"ref_verify_{name}.npz"))
    A, B, M, C, f, g = cfgs.build_problem(name)
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
    r = f.shape[1]
    st = _golden_state(gold, r)
    gap = residual_gap(prob, st)
    want = float(gold["residual_gap"])
    assert abs(gap - want) <= 1e-9 * want, (gap, want)
    fid = verify_factor_identity(prob, st)
    assert fid <= 1e-15, fid
    st.inner_residuals_A = [np.zeros_like(b) for b in st.inner_residuals_A]
    fid0 = verify_factor_identity(prob, st)
    hist = [tuple(p) for p in gold["shift_history"]]
    want0 = orc.verify_factor_identity(A, B, np.zeros_like(gold["S_A"]), gold["S_B"], gold["Z"],
                                       gold["Y"], gold["w"], gold["t"], gold["gammas"], hist, r,
                                       M=M, C=C)
    # the defect is ||S^A|| / scale plus the identity's own rounding (about
    # 1e-18 of the scale, i.e. ~1e-6 of this value)
    assert abs(fid0 - want0) <= 1e-6 * want0, (fid0, want0)


@pytest.mark.parametrize("name", ["c1", "c3s"])
def test_device_run_retains_inner_residuals(name):
    """keep_inner_residuals=True (adi.py:533-535) on the device driver: S^A and
    S^B are retained per step, the gap they give equals the oracle's on the
    downloaded blocks, it is bounded by the running estimate u + v, and the
    factor identities hold to rounding."""
    import paper_2312_02891_b200 as pb
    from paper_2312_02891_b200.verify import residual_gap, verify_factor_identity
    spec = cfgs.CONFIGS[name]
    A, B, M, C, f, g = cfgs.build_problem(name)
    pairs, cyclic = spec.load_shift_pairs()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
    cfg = pb.AdiConfig(strategy=spec.strategy, kmax=12, precond_kind_A="jacobi",
                       precond_kind_B="jacobi", keep_inner_residuals=True)
    seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible)
    assert not eng.native
    sol, rep, st = eng.run()
    k, r = rep.outer_iterations, prob.r
    SA, SB = st.S_A(), st.S_B()
    assert SA.shape == (prob.n, k * r) and SB.shape == (prob.m, k * r)
    gap = residual_gap(prob, st)
    want = orc.residual_gap(A, B, SA, SB, sol.Z, sol.Y, st.gammas, r, M=M, C=C)
    assert abs(gap - want) <= 1e-8 * want, (gap, want)
    assert gap <= (st.u + st.v) * (1 + 1e-8)
    assert verify_factor_identity(prob, st) <= 1e-13
    # the public run() returns host blocks that the host oracle accepts too
    sol2, rep2 = pb.run(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible)
    assert rep2.outer_iterations == k
