"""Row-partitioned inner solves on the GPU through the C-ABI.

The ranks of an in-process group run on one device in rank order (halo
exchange by device copies, all-reduce by a device sum, no kernel waits on
another rank's kernel), so the multi-rank algorithm is checked here against
the single-GPU engine and the oracle: SpMM identical, same iteration counts
(+-2 allowed by the contract), solutions equal to rounding.  The NCCL
communicator is exercised at world size 1 (one B200 per gpurun call)."""

import os
import socket
import warnings

import numpy as np
import pytest

from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200 import configs as cfgs

from conftest import GOLD, read_steps_csv

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x.astype(np.complex128))).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.fixture(scope="module")
def c1():
    return cfgs.build_problem("c1")


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("side", ["A", "B"])
def test_rowpart_apply_matches_single(c1, rng, P, side):
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    from paper_2312_02891_b200.rowpart import RowPartitionedGmres
    A, B = c1[0], c1[1]
    base = A if side == "A" else B
    shift = -3.5 + 1.25j
    rp = RowPartitionedGmres(side, base, None, nranks=P, restart=20)
    single = DeviceOperator(DeviceMatrix(base, transpose=(side == "B")), None, shift,
                            adjoint=(side == "B"))
    n = base.shape[0]
    x = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
    y = host(rp.apply_device(shift, dev(x)))
    want = host(single.apply(dev(x)))
    assert np.array_equal(y, want)       # same per-row order, same FMAs
    ref = orc.ShiftedOp(base, None, shift, adjoint=(side == "B")).apply(x)
    assert np.max(np.abs(y - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("P", [2, 4])
def test_rowpart_dinv_halo(c1, P):
    """Jacobi dinv of the halo rows arrives from their owners."""
    from paper_2312_02891_b200 import _lib
    from paper_2312_02891_b200.rowpart import RowPartitionedGmres
    A = c1[0]
    shift = -2.0 + 0.5j
    rp = RowPartitionedGmres("A", A, None, nranks=P)
    ops = rp.operator(shift)
    full = 1.0 / (A.diagonal() + shift)
    for pl, op in zip(rp.plans, ops):
        buf = np.zeros(2 * (pl.n_loc + pl.n_halo))
        # sad_op_get_dinv copies the n_loc local values (the halo part is
        # exercised by the solves, whose first SpMM gathers it)
        _lib.check(_lib.load().sad_op_get_dinv(op.h, buf.ctypes.data))
        loc = buf[:2 * pl.n_loc].view(np.complex128)
        assert np.allclose(loc, full[pl.r0:pl.r1], rtol=1e-15, atol=0)


@pytest.mark.parametrize("orth", ["dcgs2", "cgs2"])
@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("side,flexible", [("A", False), ("B", False), ("A", True)])
def test_rowpart_gmres_matches_single_gpu(c1, rng, P, side, flexible, orth):
    from paper_2312_02891_b200.krylov import GpuGmresBinding
    from paper_2312_02891_b200.rowpart import RowPartitionedGmres
    A, B = c1[0], c1[1]
    base = A if side == "A" else B
    n = base.shape[0]
    shift = -40.0 + 12.0j
    rhs = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
    delta = 1e-9 * np.linalg.norm(rhs)
    # the single-GPU engine with the same orthogonalisation
    one = GpuGmresBinding(side, base, None, restart=30, flexible=flexible,
                          engine="persistent" if orth == "dcgs2" else "multi")
    r1 = one.solve(shift, rhs, delta)
    rp = RowPartitionedGmres(side, base, None, nranks=P, restart=30, flexible=flexible,
                             orth=orth)
    rP = rp.solve(shift, rhs, delta)
    assert np.all(rP.converged)
    assert np.all(np.abs(rP.iterations - r1.iterations) <= 2), (rP.iterations, r1.iterations)
    scale = np.max(np.abs(r1.solution))
    assert np.max(np.abs(rP.solution - r1.solution)) <= 1e-8 * scale
    # the returned residual is the true one (krylov.py:62)
    op = orc.ShiftedOp(base, None, shift, adjoint=(side == "B"))
    true = rhs - op.apply(rP.solution)
    assert np.max(np.abs(true - rP.residual)) <= 1e-10 * np.max(np.abs(rhs))
    assert np.all(np.linalg.norm(true, axis=0) <= delta / 2 * (1 + 1e-6))


def test_rowpart_gmres_real_block_and_oracle(c1, rng):
    """fp64 block, real shift, against the oracle restatement's counts."""
    from paper_2312_02891_b200.rowpart import RowPartitionedGmres
    A = c1[0]
    n = A.shape[0]
    shift = -25.0
    rhs = rng.standard_normal((n, 3))
    delta = 1e-8 * np.linalg.norm(rhs)
    rp = RowPartitionedGmres("A", A, None, nranks=3, restart=50)
    b = torch.from_numpy(rhs).cuda()
    out = rp.solve_device(shift, b, delta)
    x = host(out.solution)
    ref = orc.Binding("A", A, None, solver="gmres", max_iterations=1000, restart=50,
                      precond="jacobi", orth="cgs2").solve(shift, rhs, delta)
    assert np.all(np.abs(out.iterations - ref.iterations) <= 2), (out.iterations, ref.iterations)
    assert np.max(np.abs(x - ref.solution)) <= 1e-7 * np.max(np.abs(ref.solution))
    res = rhs - (A @ x + shift * x)
    assert np.all(np.linalg.norm(res, axis=0) <= delta / 3 * (1 + 1e-6))


def test_rowpart_maxit_flagged(c1, rng):
    from paper_2312_02891_b200.rowpart import RowPartitionedGmres
    A = c1[0]
    rhs = rng.standard_normal((A.shape[0], 2)) + 0j
    rp = RowPartitionedGmres("A", A, None, nranks=2, restart=10, max_iterations=7)
    out = rp.solve(-1.0, rhs, 1e-14)
    assert np.all(out.iterations == 7)
    assert not np.any(out.converged)


def test_rowpart_adi_c1_matches_golden():
    """The whole config-1 ADI with both sides row-partitioned over 3 ranks:
    same outer steps as the oracle, inner counts within +-2, residual < 1e-8."""
    import paper_2312_02891_b200 as pb
    spec = cfgs.CONFIGS["c1"]
    A, B, M, C, f, g = cfgs.build_problem("c1")
    pairs, cyclic = spec.load_shift_pairs()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
    cfg = pb.AdiConfig(strategy=spec.strategy, kmax=spec.kmax,
                       outer_tolerance=spec.outer_tolerance,
                       precond_kind_A="jacobi", precond_kind_B="jacobi")
    seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                       row_ranks=3)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        sol, rep, _ = eng.run()
    gold = read_steps_csv(os.path.join(GOLD, "oracle_c1_gmres.csv"))
    assert rep.converged and rep.final_scaled_residual < 1e-8
    assert rep.outer_iterations == len(gold)
    for rec, gd in zip(rep.records, gold):
        assert abs(rec.inner_it_A - gd["inner_it_A"]) <= 2
        assert abs(rec.inner_it_B - gd["inner_it_B"]) <= 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_rowpart_nccl_world1(c1, rng):
    """NCCL communicator (dlopen'd libnccl) at world size 1: allreduce and the
    solve loop's collectives run through NCCL."""
    import torch.distributed as dist
    from paper_2312_02891_b200.rowpart import RowPartitionedGmres
    from paper_2312_02891_b200.krylov import GpuGmresBinding
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}",
                                rank=0, world_size=1)
    try:
        A = c1[0]
        rp = RowPartitionedGmres("A", A, None, nranks=1, restart=30, comm="nccl")
        t = [torch.arange(10, dtype=torch.float64, device="cuda")]
        rp.allreduce_(t)
        assert torch.equal(t[0].cpu(), torch.arange(10, dtype=torch.float64))
        rhs = rng.standard_normal((A.shape[0], 2)) + 1j * rng.standard_normal((A.shape[0], 2))
        delta = 1e-9 * np.linalg.norm(rhs)
        out = rp.solve(-40.0 + 12.0j, rhs, delta)
        one = GpuGmresBinding("A", A, None, restart=30, engine="multi").solve(-40.0 + 12.0j, rhs, delta)
        assert np.all(np.abs(out.iterations - one.iterations) <= 2)
        assert np.max(np.abs(out.solution - one.solution)) <= 1e-8 * np.max(np.abs(one.solution))
    finally:
        if own:
            dist.destroy_process_group()


@pytest.mark.parametrize("force", [False, True])
def test_sharded_adi_world1_c1(force):
    """multigpu.make_sharded at world size 1 (both sides on rank 0, NCCL
    communicators of size 1): the one-process-per-GPU driver end to end."""
    import torch.distributed as dist
    import paper_2312_02891_b200 as pb
    from paper_2312_02891_b200.multigpu import make_sharded
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}",
                                rank=0, world_size=1)
    try:
        spec = cfgs.CONFIGS["c1"]
        A, B, M, C, f, g = cfgs.build_problem("c1")
        pairs, cyclic = spec.load_shift_pairs()
        prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
        cfg = pb.AdiConfig(strategy=spec.strategy, kmax=spec.kmax,
                           outer_tolerance=spec.outer_tolerance,
                           precond_kind_A="jacobi", precond_kind_B="jacobi")
        seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
        run = make_sharded(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                           force_rowpart=force)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            factors, gammas, rep = run.run()
        gold = read_steps_csv(os.path.join(GOLD, "oracle_c1_gmres.csv"))
        assert rep.converged and rep.outer_iterations == len(gold)
        for rec, gd in zip(rep.records, gold):
            assert abs(rec.inner_it_A - gd["inner_it_A"]) <= 2
            assert abs(rec.inner_it_B - gd["inner_it_B"]) <= 2
        assert len(factors["A"]) == len(factors["B"]) == rep.outer_iterations
    finally:
        if own:
            dist.destroy_process_group()


@pytest.mark.parametrize("P", [1, 3])
@pytest.mark.parametrize("r,cplx,flexible", [(2, True, False), (3, True, True), (8, False, False), (5, False, False)])
def test_rowpart_ring_sweeps_match_direct_kernels(c1, rng, monkeypatch, P, r, cplx, flexible):
    """The DCGS2 sweeps through the TMA ring (k_dot_dual_ring / k_update_ring,
    forced here at a small size with SAD_DIST_RING=2; by default only for large
    slabs) against the direct-load kernels they replace (SAD_DIST_RING=0): same
    iteration counts, solutions to 1e-10, and the single-GPU counts (+-2)."""
    from paper_2312_02891_b200.krylov import GpuGmresBinding
    from paper_2312_02891_b200.rowpart import RowPartitionedGmres
    A = c1[0]
    n = A.shape[0]
    shift = -40.0 + (12.0j if cplx else 0.0)
    rhs = rng.standard_normal((n, r)) + (1j * rng.standard_normal((n, r)) if cplx else 0.0)
    delta = 1e-9 * np.linalg.norm(rhs)
    out = {}
    for mode in ("2", "0"):
        monkeypatch.setenv("SAD_DIST_RING", mode)
        rp = RowPartitionedGmres("A", A, None, nranks=P, restart=30, flexible=flexible)
        out[mode] = rp.solve(shift, rhs, delta)
    ring, direct = out["2"], out["0"]
    assert np.all(ring.converged)
    assert np.array_equal(ring.iterations, direct.iterations)
    assert np.max(np.abs(ring.solution - direct.solution)) <= 1e-10 * np.max(np.abs(direct.solution))
    one = GpuGmresBinding("A", A, None, restart=30, flexible=flexible).solve(shift, rhs, delta)
    assert np.all(np.abs(ring.iterations - one.iterations) <= 2)
