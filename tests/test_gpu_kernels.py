"""GPU parity of the kernels through the C-ABI, against the CPU oracle."""

import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200 import configs as cfgs

from conftest import GOLD

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def dev(x, complex_=True):
    return torch.from_numpy(np.ascontiguousarray(x.astype(np.complex128 if complex_ else np.float64))).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def rand_sparse(rng, n, density=0.3, diag=4.0):
    d = rng.standard_normal((n, n))
    d[rng.random((n, n)) > density] = 0.0
    d += np.diag(diag + rng.random(n))
    return sp.csr_matrix(d)


# -- shifted SpMM ---------------------------------------------------------------

@pytest.mark.parametrize("r", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("shift", [-1.7 + 0j, -2.0 + 0.4j])
@pytest.mark.parametrize("adjoint", [False, True])
@pytest.mark.parametrize("with_mass", [False, True])
def test_shifted_apply_matches_oracle(rng, r, shift, adjoint, with_mass):
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    n = 37
    base = rand_sparse(rng, n)
    mass = rand_sparse(rng, n) if with_mass else None
    x = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    ref = orc.ShiftedOp(base, mass, shift, adjoint=adjoint)
    dm = DeviceMatrix(base, transpose=adjoint)
    dmm = None if mass is None else DeviceMatrix(mass, transpose=adjoint)
    op = DeviceOperator(dm, dmm, shift, adjoint=adjoint)
    y = host(op.apply(dev(x)))
    want = ref.apply(x)
    # test_sparse.py:99-106 / 116-124 tolerances
    assert np.max(np.abs(y - want)) <= 1e-13 * np.max(np.abs(want))
    # residual mode
    b = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    res = host(op.residual(dev(b), dev(x)))
    assert np.max(np.abs(res - (b - want))) <= 1e-13 * np.max(np.abs(want))
    # Jacobi
    d = op.dinv()
    assert np.max(np.abs(d - orc.jacobi_dinv(ref))) <= 1e-15 * np.max(np.abs(d))
    if shift.imag == 0 and True:
        xr = rng.standard_normal((n, r))
        yr = host(op.apply(dev(xr, complex_=False)))
        assert yr.dtype == np.float64
        assert np.max(np.abs(yr - ref.apply(xr).real)) <= 1e-13 * np.max(np.abs(yr))


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_config_operators_match_oracle(rng, name):
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    A, B, M, C, f, g = cfgs.build_problem(name)
    pairs, _ = cfgs.CONFIGS[name].load_shift_pairs()
    for mat, adjoint, shift in ((A, False, pairs[0][1]), (B, True, pairs[0][0])):
        r = 3
        x = rng.standard_normal((mat.shape[0], r)) + 1j * rng.standard_normal((mat.shape[0], r))
        op = DeviceOperator(DeviceMatrix(mat, transpose=adjoint), None, shift, adjoint=adjoint)
        want = orc.ShiftedOp(mat, None, shift, adjoint=adjoint).apply(x)
        got = host(op.apply(dev(x)))
        assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


def test_plain_and_transpose_apply(rng):
    from paper_2312_02891_b200.device import DeviceMatrix
    m = sp.random(50, 30, density=0.2, random_state=3, format="csr")
    dm = DeviceMatrix(m, transpose=True)
    x = rng.standard_normal((30, 4))
    assert np.allclose(host(dm.apply(dev(x, False))), m @ x, rtol=0, atol=1e-13)
    x2 = rng.standard_normal((50, 2)) + 1j * rng.standard_normal((50, 2))
    assert np.allclose(host(dm.apply(dev(x2), transpose=True)), m.T @ x2, rtol=0, atol=1e-13)


def test_zero_diagonal_breakdown():
    from paper_2312_02891_b200 import _lib
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    m = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 2.0]]))
    with pytest.raises(_lib.FactorizationBreakdown):
        DeviceOperator(DeviceMatrix(m), None, 0.0)


def test_dimension_errors():
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    a = DeviceMatrix(sp.eye(4, format="csr"))
    b = DeviceMatrix(sp.eye(5, format="csr"))
    with pytest.raises(ValueError):
        DeviceOperator(a, b, 1.0)
    with pytest.raises(ValueError):
        DeviceOperator(a, None, 1.0, adjoint=True)   # transpose not built


# -- block utilities ----------------------------------------------------------------

@pytest.mark.parametrize("r", [1, 3, 8])
def test_gram_and_axpy(rng, r):
    from paper_2312_02891_b200.device import axpy, gram
    n = 10007
    x = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    y = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    G = gram(dev(x), dev(y))
    ref = x.conj().T @ y
    assert np.max(np.abs(G - ref)) <= 1e-12 * np.max(np.abs(ref))
    xr = rng.standard_normal((n, r))
    Gr = gram(dev(xr, False))
    assert np.max(np.abs(Gr - xr.T @ xr)) <= 1e-12 * np.max(np.abs(Gr))
    yt = dev(y)
    axpy(0.5 - 2j, dev(x), yt)
    assert np.max(np.abs(host(yt) - (y + (0.5 - 2j) * x))) <= 1e-14 * np.max(np.abs(y))


# -- GMRES solves against the oracle ---------------------------------------------------

# persistent engine with each phase-A path (auto picks "direct" at these sizes)
ENGINES = [("persistent", "dcgs2"), ("persistent-tma", "dcgs2"), ("multi", "cgs2")]


def _binding_kw(engine):
    if engine == "persistent-tma":
        return dict(engine="persistent", phase_a="tma")
    return dict(engine=engine)


def _solve_both(mat, adjoint, shift, rhs, delta, restart, flexible=False, maxit=1000,
                precond="jacobi", engine="persistent"):
    from paper_2312_02891_b200 import GpuGmresBinding
    side = "B" if adjoint else "A"
    orth = dict(ENGINES)[engine]
    gb = GpuGmresBinding(side, mat, None, precond_kind=precond, max_iterations=maxit,
                         restart=restart, flexible=flexible, **_binding_kw(engine))
    got = gb.solve(shift, rhs, delta)
    ob = orc.Binding(side, mat, None, solver="fgmres" if flexible else "gmres",
                     max_iterations=maxit, restart=restart, precond=precond, orth=orth)
    want = ob.solve(shift, rhs, delta)
    return got, want


@pytest.mark.parametrize("engine", [e for e, _ in ENGINES])
@pytest.mark.parametrize("flexible", [False, True])
@pytest.mark.parametrize("side", ["A", "B"])
def test_gmres_c1_matches_oracle(side, flexible, engine):
    A, B, _, _, f, g = cfgs.build_problem("c1")
    pairs, _ = cfgs.CONFIGS["c1"].load_shift_pairs()
    mat, rhs = (A, f) if side == "A" else (B, g)
    for (alpha, beta) in pairs[:3]:
        shift = beta if side == "A" else alpha
        for rel in (1e-3, 1e-8, 1e-11):
            delta = rel * np.linalg.norm(rhs)
            got, want = _solve_both(mat, side == "B", shift, rhs, delta, 50, flexible,
                                    engine=engine)
            assert np.all(np.abs(got.iterations - want.iterations) <= 2), \
                (shift, rel, got.iterations, want.iterations)
            assert np.array_equal(got.converged, want.converged)
            assert np.all(got.achieved_residual_norms <= delta / rhs.shape[1]) == np.all(got.converged)
            dx = np.linalg.norm(got.solution - want.solution) / np.linalg.norm(want.solution)
            assert dx <= max(10.0 * rel, 1e-9)


@pytest.mark.parametrize("engine", [e for e, _ in ENGINES])
@pytest.mark.parametrize("r", [2, 3, 5, 8])
def test_gmres_block_columns_independent(rng, r, engine):
    """Lock-step batching keeps per-column semantics."""
    A, _, _, _, _, _ = cfgs.build_problem("c1")
    rhs = rng.standard_normal((A.shape[0], r)) * np.logspace(0, 3, r)[None, :]
    delta = 1e-7 * np.linalg.norm(rhs)
    got, want = _solve_both(A, False, -700.0 + 50.0j, rhs, delta, 20, engine=engine)
    assert np.all(np.abs(got.iterations - want.iterations) <= 2)
    assert np.array_equal(got.converged, want.converged)


@pytest.mark.parametrize("engine", [e for e, _ in ENGINES])
def test_gmres_known_answers(rng, engine):
    from paper_2312_02891_b200 import GpuGmresBinding
    # identity: <= 1 iteration (test_krylov.py:15-20)
    b = rng.standard_normal((6, 1))
    gb = GpuGmresBinding("A", sp.eye(6, format="csr"), None, restart=5, **_binding_kw(engine))
    res = gb.solve(0.0, b, 1e-12)
    assert res.total_iterations <= 1 and np.max(np.abs(res.solution - b)) < 1e-12
    # loose tolerance: 0 iterations, zero solution (test_krylov.py:27-33)
    res = gb.solve(0.0, b, 10.0 * np.linalg.norm(b))
    assert res.total_iterations == 0 and np.array_equal(res.solution, np.zeros((6, 1)))
    assert np.all(res.converged)
    # achieved norms are independent recomputes (test_krylov.py:45-54)
    d = rng.standard_normal((12, 12)) + 12 * np.eye(12)
    b = rng.standard_normal((12, 3))
    gb = GpuGmresBinding("A", sp.csr_matrix(d), None, restart=10, **_binding_kw(engine))
    res = gb.solve(0.0, b, 1e-8)
    for c in range(3):
        check = np.linalg.norm(b[:, c] - d @ res.solution[:, c])
        assert abs(check - res.achieved_residual_norms[c]) <= 1e-13 * np.linalg.norm(b[:, c])
    # request validation (test_krylov.py:128-140)
    with pytest.raises(ValueError):
        gb.solve(0.0, b, 0.0)
    with pytest.raises(ValueError):
        gb.solve(0.0, np.ones((11, 1)), 1e-8)
    with pytest.raises(ValueError):
        gb.solve(0.0, np.full((12, 1), np.inf), 1e-8)


@pytest.mark.parametrize("engine", [e for e, _ in ENGINES])
def test_gmres_maxit_nonconvergence_flagged(engine):
    A, _, _, _, f, _ = cfgs.build_problem("c1")
    got, want = _solve_both(A, False, -600.0, f, 1e-14, 5, maxit=7, engine=engine)
    assert got.iterations[0] == 7 == want.iterations[0]
    assert not got.converged[0]


@pytest.mark.parametrize("engine", [e for e, _ in ENGINES])
def test_gmres_c2_complex_matches_oracle(engine):
    A, B, _, _, f, g = cfgs.build_problem("c2")
    pairs, _ = cfgs.CONFIGS["c2"].load_shift_pairs()
    alpha, beta = pairs[0]
    for mat, adjoint, shift, rhs in ((A, False, beta, f), (B, True, alpha, g)):
        delta = 1e-9 * np.linalg.norm(rhs)
        got, want = _solve_both(mat, adjoint, shift, rhs, delta, 30, flexible=True,
                                engine=engine)
        assert np.all(np.abs(got.iterations - want.iterations) <= 2)
        assert np.all(got.converged)


@pytest.mark.parametrize("max_sms", [0, 22])
@pytest.mark.parametrize("red_min", ["8192", "1", "1000000000"])
def test_persistent_direct_path_sizing_and_grid_reduction(monkeypatch, max_sms, red_min):
    """The small-slab (direct) phase A sized for two blocks per SM (default) and
    for one (SAD_DIRECT_BPS=1), on all SMs and on config 2's B-side share of 22,
    with finisher A's reduction on the whole grid always / by the default rule /
    never (SAD_DIST_RED_MIN): the same iteration counts as the oracle's run, and
    solutions equal to 1e-10 across the variants."""
    from paper_2312_02891_b200 import GpuGmresBinding
    monkeypatch.setenv("SAD_DIST_RED_MIN", red_min)
    _, B, _, _, _, g = cfgs.build_problem("c2")
    pairs, _ = cfgs.CONFIGS["c2"].load_shift_pairs()
    alpha = pairs[0][0]
    delta = 1e-9 * np.linalg.norm(g)
    want = orc.Binding("B", B, None, solver="fgmres", restart=30, orth="dcgs2").solve(alpha, g, delta)
    sols = []
    for bps in ("2", "1"):
        monkeypatch.setenv("SAD_DIRECT_BPS", bps)
        gb = GpuGmresBinding("B", B, None, precond_kind="jacobi", restart=30, flexible=True,
                             engine="persistent", phase_a="direct", max_sms=max_sms)
        got = gb.solve(alpha, g, delta)
        assert np.all(got.converged)
        assert np.all(np.abs(got.iterations - want.iterations) <= 2)
        sols.append(got.solution)
    assert np.linalg.norm(sols[0] - sols[1]) <= 1e-10 * np.linalg.norm(sols[1])
    assert np.linalg.norm(sols[0] - want.solution) <= 1e-7 * np.linalg.norm(want.solution)


@pytest.mark.parametrize("engine", [e for e, _ in ENGINES])
def test_gmres_fixed_steps_match_oracle(rng, engine):
    """Fixed-step mode (config 4 path): the true residual after 40 steps
    matches the oracle's (same Krylov space, same least-squares solution)."""
    from paper_2312_02891_b200 import GpuGmresBinding
    A = cfgs.convdiff_fd(2, 128, (100.0, 100.0))
    rhs = rng.standard_normal((A.shape[0], 8))
    gb = GpuGmresBinding("A", A, None, restart=40, **_binding_kw(engine))
    out = gb.solve_device(-5000.0, torch.from_numpy(rhs).cuda(), 1.0, fixed_steps=40)
    assert np.all(out.iterations == 40)
    ob = orc.Binding("A", A, None, solver="gmres", restart=40, max_iterations=40,
                     orth=dict(ENGINES)[engine])
    want = ob.solve(-5000.0, rhs, 1e-300 * 8)
    rel = np.abs(out.achieved_residual_norms - want.achieved_residual_norms) / want.achieved_residual_norms
    assert np.all(rel < 1e-6), rel


@pytest.mark.parametrize("engine", [e for e, _ in ENGINES])
def test_gmres_c4_fixed_steps_1024_golden(engine):
    """Config 4's path at depth: 100 fixed Jacobi-GMRES(100) steps,
    r = 8, on the config-4 operator at 1024^2 (1M rows: many tiles per block, the
    TMA ring of phase A, a 100-block basis) against the oracle's per-column true
    residual norms (tests/golden/make_golden_c4.py)."""
    from paper_2312_02891_b200 import GpuGmresBinding
    gold = np.load(os.path.join(GOLD, "oracle_c4_1024_fixed.npz"))
    n0, r, steps, shift = int(gold["n0"]), int(gold["r"]), int(gold["steps"]), float(gold["shift"])
    A, X = cfgs.build_c4(n0, r, 0)
    gb = GpuGmresBinding("A", A, None, restart=steps, **_binding_kw(engine))
    out = gb.solve_device(shift, torch.from_numpy(X).cuda(), 1.0, fixed_steps=steps)
    assert np.all(out.iterations == steps)
    want = gold[dict(ENGINES)[engine]]
    rel = np.abs(out.achieved_residual_norms - want) / want
    assert np.all(rel < 1e-6), rel


@pytest.mark.parametrize("r", [1, 2, 3, 8])
@pytest.mark.parametrize("cplx", [False, True])
def test_adi_epilogue_matches_numpy(rng, r, cplx):
    from paper_2312_02891_b200.device import adi_epilogue
    n, m = 5003, 3001
    def blk(rows):
        b = rng.standard_normal((rows, r))
        return b + 1j * rng.standard_normal((rows, r)) if cplx else b
    mz, ra, w, cy, rb, t = blk(n), blk(n), blk(n), blk(m), blk(m), blk(m)
    gam = (-2.5 + 0.75j) if cplx else -2.5
    wd, td = dev(w, cplx), dev(t, cplx)
    G = adi_epilogue(gam, dev(mz, cplx), dev(ra, cplx), wd, dev(cy, cplx), dev(rb, cplx), td)
    w2 = w + gam * mz
    t2 = t + np.conj(gam) * cy
    assert np.max(np.abs(host(wd) - w2)) <= 1e-13 * np.max(np.abs(w2))
    assert np.max(np.abs(host(td) - t2)) <= 1e-13 * np.max(np.abs(t2))
    for k, X in enumerate((ra, rb, mz, cy, w2, t2)):
        ref = X.conj().T @ X
        assert np.max(np.abs(G[k] - ref)) <= 1e-12 * np.max(np.abs(ref)), k


@pytest.mark.parametrize("r", [1, 2, 3, 8])
def test_bulk_spmm_many_tiles(rng, r):
    """Multi-tile path of the TMA-staged SpMM (double/triple buffers cycle)."""
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    A = cfgs.convdiff_fd(2, 300, (30.0, -20.0))     # 90k rows -> many 256-row tiles
    x = rng.standard_normal((A.shape[0], r))
    op = DeviceOperator(DeviceMatrix(A), None, -7.5 + 0j)
    y = host(op.apply(dev(x, False)))
    want = A @ x - 7.5 * x
    assert np.max(np.abs(y - want)) <= 1e-13 * np.max(np.abs(want))
    xc = x + 1j * rng.standard_normal(x.shape)
    op2 = DeviceOperator(DeviceMatrix(A, transpose=True), None, -3.0 + 2.0j, adjoint=True)
    y2 = host(op2.apply(dev(xc)))
    want2 = A.T @ xc + np.conj(-3.0 + 2.0j) * xc
    assert np.max(np.abs(y2 - want2)) <= 1e-13 * np.max(np.abs(want2))


def test_allocation_cache_reuse_and_trim(rng):
    """Device buffers of destroyed handles are reused (sad_capi.cu DevCache):
    operators built in the memory of destroyed ones give the same results,
    and sad_ctx_trim releases the cache."""
    import gc
    from paper_2312_02891_b200 import _lib
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    n, r = 211, 3
    base = rand_sparse(rng, n)
    mass = rand_sparse(rng, n)
    x = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    shifts = [-1.5 + 0.3j, -2.5 - 0.1j, -0.75 + 0.0j]
    want = [orc.ShiftedOp(base, mass, s).apply(x) for s in shifts]
    for round_ in range(3):
        dm = DeviceMatrix(base)
        dmm = DeviceMatrix(mass)
        ops = [DeviceOperator(dm, dmm, s) for s in shifts]
        for op, w in zip(ops, want):
            y = host(op.apply(dev(x)))
            assert np.max(np.abs(y - w)) <= 1e-13 * np.max(np.abs(w)), round_
        del ops, dm, dmm
        gc.collect()
    ctx = _lib.context(0)
    _lib.check(_lib.load().sad_ctx_trim(ctx), ctx)
    op = DeviceOperator(DeviceMatrix(base), DeviceMatrix(mass), shifts[0])
    y = host(op.apply(dev(x)))
    assert np.max(np.abs(y - want[0])) <= 1e-13 * np.max(np.abs(want[0]))
