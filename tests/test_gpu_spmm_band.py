"""The banded-plan shifted SpMM (k_spmm_band: x rows of every 64-row tile staged
in shared memory by TMA, 16-bit local column indices, padded slot-major
values) against the oracle's ShiftedOp.apply (sparse.py:192-206) and, bit for
bit, against the CSR kernel it replaces on the same operator.  The plan is
forced with SAD_SPMM_BAND=1 (by default only operators with >= 2^20 nonzeros
get one)."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200 import configs as cfgs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def dev(a, complex_=True):
    t = torch.from_numpy(np.ascontiguousarray(a if complex_ else np.asarray(a, dtype=np.float64)))
    return t.cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _ops(monkeypatch, base, mass, shift, adjoint, precond="none"):
    """The same operator with and without a banded plan."""
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    out = []
    for flag in ("1", "0"):
        monkeypatch.setenv("SAD_SPMM_BAND", flag)
        dm = DeviceMatrix(base, transpose=adjoint)
        dmm = None if mass is None else DeviceMatrix(mass, transpose=adjoint)
        out.append(DeviceOperator(dm, dmm, shift, adjoint=adjoint, precond_kind=precond))
    return out


def fd2(n0, wind=30.0):
    from paper_2312_02891_b200.problems import convdiff_fd
    return convdiff_fd(2, n0, (wind, 0.5 * wind))


@pytest.mark.parametrize("r", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("shift", [-1.7 + 0j, -2.0 + 0.4j])
@pytest.mark.parametrize("adjoint", [False, True])
def test_band_apply_matches_oracle_and_csr_kernel(monkeypatch, rng, r, shift, adjoint):
    base = fd2(37)          # n = 1369: 22 tiles, the last one partial
    n = base.shape[0]
    band, plain = _ops(monkeypatch, base, None, shift, adjoint)
    info = band.band_info()
    assert info is not None and plain.band_info() is None
    assert info["tiles"] == -(-n // info["rows"]) and info["nnz"] == base.nnz and info["wmax"] == 5
    assert info["entries"] < 1.2 * base.nnz
    x = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    want = orc.ShiftedOp(base, None, shift, adjoint=adjoint).apply(x)
    got = host(band.apply(dev(x)))
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))
    assert np.array_equal(got, host(plain.apply(dev(x))))      # same products, same order
    b = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    res = host(band.residual(dev(b), dev(x)))
    assert np.array_equal(res, host(plain.residual(dev(b), dev(x))))
    assert np.max(np.abs(res - (b - want))) <= 1e-13 * np.max(np.abs(want))
    if shift.imag == 0:
        xr = rng.standard_normal((n, r))
        yr = host(band.apply(dev(xr, complex_=False)))
        assert yr.dtype == np.float64
        assert np.array_equal(yr, host(plain.apply(dev(xr, complex_=False))))
        assert np.max(np.abs(yr - orc.ShiftedOp(base, None, shift, adjoint=adjoint).apply(xr).real)) \
            <= 1e-13 * np.max(np.abs(yr))


@pytest.mark.parametrize("r", [2, 3, 8])
@pytest.mark.parametrize("shift", [-45.0 + 0j, -45.0 + 10.0j])
@pytest.mark.parametrize("adjoint", [False, True])
def test_band_generalised_pencil(monkeypatch, rng, r, shift, adjoint):
    """base + shift*mass assembled on the merged pattern (9-point FEM pencil:
    three ranges per tile, W = 9), real and complex values."""
    from paper_2312_02891_b200.problems import fem_q1_2d
    K, M = fem_q1_2d(30, (30.0, 15.0))
    n = K.shape[0]
    band, plain = _ops(monkeypatch, K, M, shift, adjoint)
    info = band.band_info()
    assert info is not None and info["wmax"] == 9
    x = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    want = orc.ShiftedOp(K, M, shift, adjoint=adjoint).apply(x)
    got = host(band.apply(dev(x)))
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))
    assert np.array_equal(got, host(plain.apply(dev(x))))


def test_band_3d_and_irregular_patterns(monkeypatch, rng):
    """7-point 3-D stencil (five ranges per tile); a pattern with far random
    columns gets no plan and runs the CSR kernel."""
    from paper_2312_02891_b200.problems import convdiff_fd
    A = convdiff_fd(3, 14, (20.0, 20.0, 20.0))
    band, plain = _ops(monkeypatch, A, None, -3.0, False)
    assert band.band_info() is not None
    x = rng.standard_normal((A.shape[0], 4)) + 1j * rng.standard_normal((A.shape[0], 4))
    assert np.array_equal(host(band.apply(dev(x))), host(plain.apply(dev(x))))
    R = sp.random(3000, 3000, density=0.004, random_state=5, format="csr") + 4.0 * sp.eye(3000, format="csr")
    rb, rplain = _ops(monkeypatch, sp.csr_matrix(R), None, -1.0, False)
    assert rb.band_info() is None
    xr = rng.standard_normal((3000, 3)) + 0j
    want = orc.ShiftedOp(sp.csr_matrix(R), None, -1.0).apply(xr)
    assert np.max(np.abs(host(rb.apply(dev(xr))) - want)) <= 1e-13 * np.max(np.abs(want))


@pytest.mark.parametrize("engine", ["multi", "persistent", "persistent-tma"])
@pytest.mark.parametrize("flexible", [False, True])
@pytest.mark.parametrize("r,cplx", [(3, True), (8, False), (4, True), (1, False)])
def test_gmres_with_band_plan_matches_csr_path(monkeypatch, rng, engine, flexible, r, cplx):
    """Jacobi-GMRES through the banded SpMM (Jacobi prologue from the staged dinv
    rows, Arnoldi-mode scaling, FGMRES Z) -- the stand-alone kernel in the
    multi-kernel engine, the SpMM sub-phase inside the persistent kernel
    ("persistent-tma": its large-slab path) -- identical iteration counts and
    solutions to 1e-10 against the same solve on the CSR kernels."""
    from paper_2312_02891_b200 import GpuGmresBinding
    A = fd2(48, 60.0)
    n = A.shape[0]
    b = rng.standard_normal((n, r)) + (1j * rng.standard_normal((n, r)) if cplx else 0.0)
    shift = -250.0 + (90.0j if cplx else 0.0)
    out = []
    eng, _, pa = engine.partition("-")
    for flag in ("1", "0"):
        monkeypatch.setenv("SAD_SPMM_BAND", flag)
        gb = GpuGmresBinding("A", A, None, precond_kind="jacobi", restart=30, flexible=flexible,
                             engine=eng, phase_a=pa or "auto")
        cls = 1 if eng == "persistent" else 0
        info = gb.operator(shift).band_info(cls)
        assert (info is not None) == (flag == "1")
        out.append(gb.solve(shift, b, 1e-8))
    got, ref = out
    assert np.array_equal(got.iterations, ref.iterations)
    assert np.all(got.converged)
    assert np.linalg.norm(got.solution - ref.solution) <= 1e-10 * np.linalg.norm(ref.solution)
    if r <= 3:
        orc_res = orc.Binding("A", A, None, solver="fgmres" if flexible else "gmres", restart=30,
                              orth="dcgs2" if eng == "persistent" else "cgs2").solve(shift, b, 1e-8)
        assert np.all(np.abs(got.iterations - orc_res.iterations) <= 2)


@pytest.mark.parametrize("n", [1, 5, 64, 128, 257])
def test_band_edge_sizes_and_patterns(monkeypatch, rng, n):
    """Tiny and tile-aligned sizes, an empty row, a missing diagonal entry (the
    tile's own rows are staged anyway: the shift term needs them)."""
    d = rng.standard_normal((n, n))
    d[np.abs(np.subtract.outer(np.arange(n), np.arange(n))) > 2] = 0.0      # pentadiagonal
    if n >= 5:
        d[3, :] = 0.0            # empty row
        d[1, 1] = 0.0            # no diagonal entry in row 1
    A = sp.csr_matrix(d)
    A.eliminate_zeros()
    for shift in (-0.7 + 0j, 0.3 - 1.1j):
        band, plain = _ops(monkeypatch, A, None, shift, False)
        assert band.band_info() is not None
        for r in (1, 3, 8):
            x = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
            want = orc.ShiftedOp(A, None, shift).apply(x)
            got = host(band.apply(dev(x)))
            assert np.array_equal(got, host(plain.apply(dev(x))))
            assert np.max(np.abs(got - want)) <= 1e-13 * max(np.max(np.abs(want)), 1e-300)


@pytest.mark.parametrize("rows", ["32", "64", "128", "256"])
def test_band_tile_rows_override(monkeypatch, rng, rows):
    """SAD_BAND_ROWS: every tile size gives the CSR kernel's bits (the 3-D stencil
    needs five ranges per tile; 256-row tiles merge the +-n0 ranges)."""
    from paper_2312_02891_b200.problems import convdiff_fd
    monkeypatch.setenv("SAD_BAND_ROWS", rows)
    A = convdiff_fd(3, 12, (20.0, -20.0, 20.0))
    band, plain = _ops(monkeypatch, A, None, -3.0 + 2.0j, True)
    info = band.band_info()
    assert info is not None and info["rows"] == int(rows)
    x = rng.standard_normal((A.shape[0], 4)) + 1j * rng.standard_normal((A.shape[0], 4))
    assert np.array_equal(host(band.apply(dev(x))), host(plain.apply(dev(x))))
