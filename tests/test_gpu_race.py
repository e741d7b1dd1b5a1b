"""Race stress of the persistent GMRES kernel's redundant phase-C finisher.

Every block forms the step's Givens rotation itself after the phase-C barrier,
while block 0 alone writes the global state (active flags, iteration counts,
g).  SAD_OPT_DEBUG_DELAY makes the LAST block idle after every phase-C release,
so block 0 has long rewritten that state before the late block's finisher runs:
the solve must still be bit-identical to an undelayed one (each block keeps
its own copy of the per-column state)."""

import numpy as np
import pytest

from paper_2312_02891_b200 import GpuGmresBinding, _lib
from paper_2312_02891_b200 import configs as cfgs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _solve(gb, shift, rhs, delta, delay_ns):
    dtype = _lib.SAD_C128 if rhs.dtype == torch.complex128 else _lib.SAD_F64
    ws = gb.workspace(rhs.shape[1], dtype)
    ws.set_option(_lib.SAD_OPT_DEBUG_DELAY, delay_ns)
    try:
        out = gb.solve_device(shift, rhs, delta)
        torch.cuda.synchronize()
    finally:
        ws.set_option(_lib.SAD_OPT_DEBUG_DELAY, 0)
    return out.iterations.copy(), out.solution.cpu().numpy(), out.achieved_residual_norms.copy()


@pytest.mark.parametrize("phase_a", ["direct", "tma"])
@pytest.mark.parametrize("name,restart", [("c1", 50), ("c2", 30)])
def test_late_block_sees_its_own_givens_state(name, restart, phase_a):
    A, B, M, C, f, g = cfgs.build_problem(name)
    pairs, _ = cfgs.CONFIGS[name].load_shift_pairs()
    beta = complex(pairs[1][1])
    gb = GpuGmresBinding("A", A, M, precond_kind="jacobi", restart=restart, phase_a=phase_a,
                         max_iterations=400)
    rhs = torch.from_numpy(np.ascontiguousarray(f.astype(np.complex128))).cuda()
    # a tight target: several restart cycles and columns ending at different steps
    delta = 1e-10 * float(np.linalg.norm(f))
    it0, x0, n0 = _solve(gb, beta, rhs, delta, 0)
    it1, x1, n1 = _solve(gb, beta, rhs, delta, 200_000)   # 200 us per step
    assert it0.tolist() == it1.tolist()
    assert np.array_equal(x0, x1)
    assert np.array_equal(n0, n1)
    assert int(it0.max()) > restart    # at least one restart happened
