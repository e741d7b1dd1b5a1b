"""The A || B split with the DEVICE side ops: rank 0 solves the
A side and rank 1 the B side with libsylvadi_b200 kernels, exchanging only the
O(r^2) Gram matrices per outer step.  This pod has one GPU, so both ranks
share cuda:0 -- a functional check of the device path (their kernels never
wait on each other; the exchange is a host all_gather over gloo), not a
scaling measurement.  Reference: the single-process device driver."""

import os
import socket
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        from paper_2312_02891_b200 import GpuGmresBinding
        from paper_2312_02891_b200 import configs as cfgs
        from paper_2312_02891_b200.adi import AdiConfig
        from paper_2312_02891_b200.parallel import Comm, DeviceSideOps, SideSplitAdi
        from paper_2312_02891_b200.shifts import ShiftSequence
        torch.cuda.set_device(0)
        spec = cfgs.CONFIGS["c1"]
        A, B, M, C, f, g = cfgs.build_problem("c1")
        pairs, cyclic = spec.load_shift_pairs()
        side = "A" if rank == 0 else "B"
        bind = GpuGmresBinding(side, A if side == "A" else B, None, restart=spec.restart)

        def solver(shift, rhs, delta):
            res = bind.solve_device(shift, rhs, delta)
            return res.solution, res.residual, res.iterations, res.converged

        cfg = AdiConfig(strategy=spec.strategy, kmax=spec.kmax)
        rhs = (f if side == "A" else g).astype(complex)
        run = SideSplitAdi(Comm(), side, solver, DeviceSideOps(), rhs, cfg,
                           ShiftSequence(pairs=pairs, cyclic=cyclic))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            factors, gammas, rep = run.run()
        np.savez(out_path + f".{rank}.npz", it_a=[r.inner_it_A for r in rep.records],
                 it_b=[r.inner_it_B for r in rep.records],
                 res=[r.scaled_res for r in rep.records], steps=rep.outer_iterations,
                 converged=rep.converged,
                 factor=torch.cat(factors, dim=1).cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_side_split_device_matches_single_process(tmp_path):
    import paper_2312_02891_b200 as pb
    from paper_2312_02891_b200 import configs as cfgs
    out = str(tmp_path / "split")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    g0, g1 = np.load(out + ".0.npz"), np.load(out + ".1.npz")
    spec = cfgs.CONFIGS["c1"]
    A, B, M, C, f, g = cfgs.build_problem("c1")
    pairs, cyclic = spec.load_shift_pairs()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
    cfg = pb.AdiConfig(strategy=spec.strategy, kmax=spec.kmax)
    sol, rep = pb.run(prob, cfg, pb.ShiftSequence(pairs=pairs, cyclic=cyclic),
                      restart=spec.restart)
    for got in (g0, g1):        # both ranks hold the same (replicated) report
        assert bool(got["converged"]) and int(got["steps"]) == rep.outer_iterations
        assert np.all(np.abs(np.array(got["it_a"]) - [r.inner_it_A for r in rep.records]) <= 2)
        assert np.all(np.abs(np.array(got["it_b"]) - [r.inner_it_B for r in rep.records]) <= 2)
    # rank 0 holds Z, rank 1 holds Y: the factors equal the single-process ones
    rel_z = np.linalg.norm(g0["factor"] - sol.Z) / np.linalg.norm(sol.Z)
    rel_y = np.linalg.norm(g1["factor"] - sol.Y) / np.linalg.norm(sol.Y)
    assert rel_z < 1e-6 and rel_y < 1e-6, (rel_z, rel_y)
