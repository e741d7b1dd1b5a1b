"""The hot path at BASELINE.json's FULL sizes, checked through properties that do
not need a second full-size solver run: the oracle's apply on the whole
config-4 block (one CPU SpMM), linearity, the adjoint identity, bit identity of
the banded plan with the CSR kernel, the GMRES recurrence against an
independently computed true residual, and -- on config 3 at 1000^2 / 700^2 --
the ADI factor identities and the residual-gap bound of adi.py:632-679.

The small-size parity tests (oracle runs, golden vectors) are in
test_gpu_kernels.py / test_gpu_spmm_band.py / test_gpu_adi.py; these cases make
sure nothing changes where the tiles, the TMA rings and the 32-bit offsets are
at the sizes the metric is quoted on (n = 16.7M rows, 84M nonzeros, 1.07 GB
blocks)."""

import json
import os

import numpy as np
import pytest

from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200 import configs as cfgs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


@pytest.fixture(scope="module")
def c4():
    """Config 4 as bench.py runs it: 4096^2 grid, r = 8, the pinned shift."""
    with open(os.path.join(REPO, "configs", "shift_c4.json")) as fh:
        d = json.load(fh)
    n0 = int(d["n0"])
    assert n0 == 4096
    A, X = cfgs.build_c4(n0=n0, r=8, seed=0)
    return A, X, float(d["shift"])


def _rel(a, b):
    return float(torch.linalg.norm(a - b) / torch.linalg.norm(b))


def test_c4_full_size_spmm(c4, monkeypatch):
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    A, X, shift = c4
    n, r = X.shape
    assert n == 4096 * 4096 and A.nnz == 83869696
    monkeypatch.setenv("SAD_SPMM_BAND", "0")
    plain = DeviceOperator(DeviceMatrix(A), None, shift, precond_kind="none")
    monkeypatch.delenv("SAD_SPMM_BAND")
    band = DeviceOperator(DeviceMatrix(A), None, shift, precond_kind="none")
    adj = DeviceOperator(DeviceMatrix(A, transpose=True), None, shift, adjoint=True,
                         precond_kind="none")
    x = torch.from_numpy(X).cuda()
    y = band.apply(x)
    info = band.band_info()
    assert info is not None and info["nnz"] == A.nnz and plain.band_info() is None
    assert info["tiles"] == -(-n // info["rows"])
    # the oracle's ShiftedOp.apply (sparse.py:192-206) on the whole block
    want = orc.ShiftedOp(A, None, shift).apply(X)
    got = y.cpu().numpy()
    assert np.max(np.abs(got - want.real)) <= 1e-13 * np.max(np.abs(want))
    del want, got
    # same products in the same order as the CSR kernel: identical bits
    assert torch.equal(y, plain.apply(x))
    # linearity
    g = torch.Generator(device="cuda").manual_seed(5)
    z = torch.randn((n, r), dtype=torch.float64, device="cuda", generator=g)
    lin = band.apply(2.0 * x - 3.0 * z)
    assert _rel(lin, 2.0 * y - 3.0 * band.apply(z)) <= 1e-13
    # adjoint identity <Op x, z> = <x, Op^H z> per column
    lhs = (y * z).sum(dim=0)
    rhs = (x * adj.apply(z)).sum(dim=0)
    scale = torch.linalg.norm(y, dim=0) * torch.linalg.norm(z, dim=0)
    assert float(torch.max(torch.abs(lhs - rhs) / scale)) <= 1e-13
    # complex block through the same plan: real and imaginary parts separately
    xc = torch.complex(x, z)
    yc = band.apply(xc)
    assert _rel(yc.real, y) <= 1e-14 and _rel(yc.imag, band.apply(z)) <= 1e-14
    # the host-buffer entry point (sad_op_apply_host) returns the device result
    yh = band.apply_host(X)
    assert np.array_equal(yh, y.cpu().numpy())


@pytest.mark.parametrize("engine", ["persistent", "multi"])
def test_c4_full_size_gmres_recurrence_vs_true_residual(c4, engine):
    """40 fixed Jacobi-GMRES steps on the full config-4 block: the residual
    norms the solver reports equal ||b - Op x|| computed by an independent
    apply of the operator, the residual block it returns is that residual, the
    norms fall, and both engines (delayed-Gram CGS2 in one launch / CGS2 with one
    kernel per phase) agree."""
    from paper_2312_02891_b200 import GpuGmresBinding
    A, X, shift = c4
    steps = 40
    gb = GpuGmresBinding("A", A, None, precond_kind="jacobi", restart=steps, engine=engine)
    b = torch.from_numpy(X).cuda()
    out = gb.solve_device(shift, b, 1.0, fixed_steps=steps)
    assert np.all(out.iterations == steps)
    op = gb.operator(shift)
    true_res = b - op.apply(out.solution)
    tn = torch.linalg.norm(true_res, dim=0).cpu().numpy()
    bn = torch.linalg.norm(b, dim=0).cpu().numpy()
    assert np.all(np.abs(out.achieved_residual_norms - tn) <= 1e-9 * tn)
    assert _rel(out.residual, true_res) <= 1e-9
    assert np.all(tn < 0.5 * bn)
    test_c4_full_size_gmres_recurrence_vs_true_residual.norms[engine] = tn
    other = test_c4_full_size_gmres_recurrence_vs_true_residual.norms.get(
        "multi" if engine == "persistent" else "persistent")
    if other is not None:
        assert np.all(np.abs(tn - other) <= 1e-6 * other)


test_c4_full_size_gmres_recurrence_vs_true_residual.norms = {}


def test_c3_full_size_factor_identities_and_gap():
    """Config 3 at full size (generalised Q1-FEM pencils 1000^2 / 700^2, r = 3,
    complex shifts), four outer steps with the inner residual blocks retained:
    the factored residual identity of every step holds to rounding
    (verify_factor_identity, adi.py:655-679), the residual gap is inside the
    running budget u + v (adi.py:632-653), and the true residual of the
    downloaded factors (power iteration on the device: a lower estimate of the
    spectral norm, slow to converge on the three close singular values of an
    r = 3 residual) is below the reported low-rank residual plus that gap and
    within 1 % of it."""
    import paper_2312_02891_b200 as pb
    from paper_2312_02891_b200.verify import (residual_gap, true_residual_norm,
                                               verify_factor_identity)
    spec = cfgs.CONFIGS["c3"]
    A, B, M, C, f, g = cfgs.build_problem("c3")
    assert A.shape[0] == 1000 * 1000 and B.shape[0] == 700 * 700
    pairs, cyclic = spec.load_shift_pairs()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
    cfg = pb.AdiConfig(strategy=spec.strategy, kmax=4, precond_kind_A="jacobi",
                       precond_kind_B="jacobi", keep_inner_residuals=True)
    eng = pb.DeviceAdi(prob, cfg, pb.ShiftSequence(pairs=pairs, cyclic=cyclic),
                       restart=spec.restart, flexible=spec.flexible)
    sol, rep, st = eng.run()
    assert rep.outer_iterations == 4 and not rep.converged
    # (an inner solve may stop at max_inner_iterations here, as in the reference's
    # run of this config: the gap uses the ACHIEVED residuals, so the bounds hold)
    assert verify_factor_identity(prob, st) <= 1e-12
    gap = residual_gap(prob, st)
    assert gap <= (st.u + st.v) * (1 + 1e-8)
    reported = rep.final_scaled_residual * rep.rhs_norm
    true = true_residual_norm(prob, sol)
    assert true <= (reported + gap) * (1 + 1e-9), (true, reported, gap)
    assert true >= 0.99 * reported, (true, reported, gap)


def test_c5_full_size_spmm_and_inner_solve(monkeypatch, rng):
    """Config 5's A side at full size (3-D conv-diff, 200^3 = 8M rows, r = 4,
    complex128, the first pinned shift pair): the banded SpMM against the oracle's
    apply and, bit for bit, the CSR kernel; one Jacobi-GMRES(30) inner solve to a
    relative 1e-6 meets its per-column target in the TRUE residual."""
    from paper_2312_02891_b200 import GpuGmresBinding
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    spec = cfgs.CONFIGS["c5"]
    A = cfgs.build_problem("c5")[0]
    n, r = A.shape[0], 4
    assert n == 200 ** 3
    pairs, _ = spec.load_shift_pairs()
    shift = complex(pairs[0][0])
    X = rng.standard_normal((n, r)) + 1j * rng.standard_normal((n, r))
    x = torch.from_numpy(X).cuda()
    monkeypatch.setenv("SAD_SPMM_BAND", "0")
    plain = DeviceOperator(DeviceMatrix(A), None, shift, precond_kind="none")
    monkeypatch.delenv("SAD_SPMM_BAND")
    band = DeviceOperator(DeviceMatrix(A), None, shift, precond_kind="none")
    y = band.apply(x)
    assert band.band_info() is not None and plain.band_info() is None
    assert torch.equal(y, plain.apply(x))
    want = orc.ShiftedOp(A, None, shift).apply(X)
    assert np.max(np.abs(y.cpu().numpy() - want)) <= 1e-13 * np.max(np.abs(want))
    del want, plain, band
    gb = GpuGmresBinding("A", A, None, precond_kind="jacobi", restart=spec.restart)
    bn = float(torch.linalg.norm(x))
    delta = 1e-6 * bn
    out = gb.solve_device(shift, x, delta)
    assert np.all(out.converged)
    true_res = x - gb.operator(shift).apply(out.solution)
    tn = torch.linalg.norm(true_res, dim=0).cpu().numpy()
    assert np.all(tn <= delta / r * (1 + 1e-6))
    assert np.all(np.abs(out.achieved_residual_norms - tn) <= 1e-8 * tn)
