"""sad_op_apply_host (the reference-facing ShiftedOperator.apply with host
blocks, sparse.py:192-206): chunked, pipelined upload / SpMM / download must
equal the device-resident apply bit for bit, and the oracle to 1e-13."""

import numpy as np
import pytest

from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200 import configs as cfgs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _ops(mat, mass, shift, adjoint):
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    dm = DeviceMatrix(mat, transpose=adjoint)
    dmm = None if mass is None else DeviceMatrix(mass, transpose=adjoint)
    return DeviceOperator(dm, dmm, shift, adjoint=adjoint, precond_kind="none")


@pytest.mark.parametrize("pinned", [True, False])
def test_apply_host_config4_family_multi_chunk(pinned):
    # 1024^2 grid, r = 8 fp64: a 64 MiB block, several pipelined chunks
    A, X = cfgs.build_c4(n0=1024, r=8, seed=3)
    shift = -0.1 * 8.0 * 1025.0 ** 2
    op = _ops(A, None, shift, False)
    if pinned:
        xh = torch.empty(X.shape, dtype=torch.float64, pin_memory=True)
        xh.copy_(torch.from_numpy(X))
        x = xh.numpy()
        yh = torch.empty(X.shape, dtype=torch.float64, pin_memory=True)
        out = op.apply_host(x, yh.numpy())
    else:
        x = np.ascontiguousarray(X)
        out = op.apply_host(x)
    ydev = op.apply(torch.from_numpy(X).cuda()).cpu().numpy()
    assert np.array_equal(out, ydev)
    want = orc.ShiftedOp(A, None, shift).apply(X)
    assert np.max(np.abs(out - want.real)) <= 1e-13 * np.max(np.abs(want))
    # repeated calls reuse the staging (and must not race with the last one)
    out2 = op.apply_host(x)
    assert np.array_equal(out2, ydev)


@pytest.mark.parametrize("adjoint", [False, True])
def test_apply_host_complex_pencil(rng, adjoint):
    A, B, M, C, f, g = cfgs.build_problem("c3s")
    shift = -3.0 + 1.5j
    op = _ops(A, M, shift, adjoint)
    x = rng.standard_normal((A.shape[0], 3)) + 1j * rng.standard_normal((A.shape[0], 3))
    out = op.apply_host(np.ascontiguousarray(x))
    want = orc.ShiftedOp(A, M, shift, adjoint=adjoint).apply(x)
    assert np.max(np.abs(out - want)) <= 1e-13 * np.max(np.abs(want))
    ydev = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(out, ydev)


def test_apply_host_rejects_bad_blocks():
    A, X = cfgs.build_c4(n0=32, r=2, seed=0)
    op = _ops(A, None, -1.0, False)
    with pytest.raises(ValueError):
        op.apply_host(np.asfortranarray(X))
    with pytest.raises(ValueError):
        op.apply_host(X[:-1].copy())
    opc = _ops(A, None, -1.0 + 1.0j, False)
    with pytest.raises(ValueError):
        opc.apply_host(np.ascontiguousarray(X))      # complex shift needs complex128
