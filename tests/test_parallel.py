"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU layer:
A || B across ranks, row partition + halo exchange, distributed block dots,
and a row-partitioned GMRES built from them (compared with the oracle)."""

import os
import socket
import warnings

import numpy as np
import pytest
import scipy.sparse as sp

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)


# -- numpy backends injected into the product's parallel layer (test side) ---------

class NumpyOps:
    def __init__(self, mass=None):
        self.mass = mass

    def copy(self, b):
        return np.array(b, dtype=complex)

    def gram(self, x):
        return x.conj().T @ x

    def apply_mass(self, x):
        return x if self.mass is None else self.mass @ x

    def epilogue_half(self, gam, mz, res, w):
        w += gam * mz
        return res.conj().T @ res, mz.conj().T @ mz, w.conj().T @ w


def _side_worker(rank, world, port, out_path):
    _init(rank, world, port)
    try:
        from oracle import sylvadi_oracle as orc
        from paper_2312_02891_b200 import configs as cfgs
        from paper_2312_02891_b200.adi import AdiConfig
        from paper_2312_02891_b200.parallel import Comm, SideSplitAdi
        from paper_2312_02891_b200.shifts import ShiftSequence
        spec = cfgs.CONFIGS["c1"]
        A, B, M, C, f, g = cfgs.build_problem("c1")
        pairs, cyclic = spec.load_shift_pairs()
        side = "A" if rank == 0 else "B"
        bind = orc.Binding(side, A if side == "A" else B, None, restart=spec.restart,
                           orth="dcgs2")

        def solver(shift, rhs, delta):
            res = bind.solve(shift, rhs, delta)
            return res.solution, res.residual, res.iterations, res.converged

        cfg = AdiConfig(strategy=spec.strategy, kmax=spec.kmax)
        run = SideSplitAdi(Comm(), side, solver, NumpyOps(),
                           f if side == "A" else g, cfg, ShiftSequence(pairs=pairs, cyclic=cyclic))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            factors, gammas, rep = run.run()
        if rank == 0:
            np.savez(out_path, it_a=[r.inner_it_A for r in rep.records],
                     it_b=[r.inner_it_B for r in rep.records],
                     res=[r.scaled_res for r in rep.records], steps=rep.outer_iterations)
    finally:
        dist.destroy_process_group()


def test_side_split_adi_matches_single_process(tmp_path):
    """A on rank 0, B on rank 1, O(r^2) exchange per step: same outer steps and
    per-step inner counts as the single-process oracle driver."""
    from oracle import sylvadi_oracle as orc
    from paper_2312_02891_b200 import configs as cfgs
    out = str(tmp_path / "side.npz")
    mp.spawn(_side_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    spec = cfgs.CONFIGS["c1"]
    A, B, M, C, f, g = cfgs.build_problem("c1")
    pairs, cyclic = spec.load_shift_pairs()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = orc.run_adi(A, B, f, g, orc.Config(strategy=spec.strategy, kmax=spec.kmax), pairs,
                          orc.Binding("A", A, None, restart=50, orth="dcgs2"),
                          orc.Binding("B", B, None, restart=50, orth="dcgs2"), cyclic=cyclic)
    assert int(got["steps"]) == ref.outer_iterations == 91
    assert list(got["it_a"]) == [r.inner_it_A for r in ref.records]
    assert list(got["it_b"]) == [r.inner_it_B for r in ref.records]
    np.testing.assert_allclose(got["res"], [r.scaled_res for r in ref.records], rtol=1e-9)


# -- row partition ------------------------------------------------------------------------

def test_row_partition_balances_nnz():
    from paper_2312_02891_b200 import configs as cfgs
    from paper_2312_02891_b200.parallel import HaloPlan, RowPartition
    A, *_ = cfgs.build_problem("c2")
    for nr in (1, 2, 4, 8):
        part = RowPartition(A.indptr, nr)
        assert part.bounds[0] == 0 and part.bounds[-1] == A.shape[0]
        sizes = [A.indptr[part.bounds[q + 1]] - A.indptr[part.bounds[q]] for q in range(nr)]
        assert max(sizes) - min(sizes) <= 2 * 7
        for q in range(nr):
            plan = HaloPlan(A, part, q)
            # 7-point stencil on 40^3, slabs along the slowest axis: one 40x40
            # neighbour plane per internal face
            faces = (q > 0) + (q < nr - 1)
            assert plan.nhalo <= faces * 40 * 40 + 2 * 40 * 40


def _halo_worker(rank, world, port, out_path):
    _init(rank, world, port)
    try:
        from paper_2312_02891_b200 import configs as cfgs
        from paper_2312_02891_b200.parallel import Comm, HaloPlan, RowPartition, halo_exchange
        A, B, *_ = cfgs.build_problem("c2")
        comm = Comm()
        part = RowPartition(A.indptr, world)
        plan = HaloPlan(A, part, rank)
        gen = np.random.default_rng(5)
        X = gen.standard_normal((A.shape[0], 3)) + 1j * gen.standard_normal((A.shape[0], 3))
        xl = torch.from_numpy(X[plan.r0:plan.r1].copy())
        xe = halo_exchange(xl, plan, comm).numpy()
        yl = plan.local_csr @ xe
        # distributed block dots: per-rank partials allreduced
        part_dot = X[plan.r0:plan.r1].conj().T @ yl
        dots = comm.allreduce_sum(part_dot)
        ys = comm.allgather(np.ascontiguousarray(
            np.pad(yl, ((0, A.shape[0] - yl.shape[0]), (0, 0)))))
        if rank == 0:
            y = np.concatenate([ys[q][:part.range(q)[1] - part.range(q)[0]]
                                for q in range(world)])
            np.savez(out_path, y=y, dots=dots, X=X)
    finally:
        dist.destroy_process_group()


def test_halo_spmm_and_dots_match_global(tmp_path):
    from paper_2312_02891_b200 import configs as cfgs
    out = str(tmp_path / "halo.npz")
    mp.spawn(_halo_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    A, *_ = cfgs.build_problem("c2")
    y_ref = A @ got["X"]
    # same per-row summation order as the global CSR: bitwise equal
    assert np.array_equal(got["y"], y_ref)
    dots_ref = got["X"].conj().T @ y_ref
    assert np.max(np.abs(got["dots"] - dots_ref)) <= 1e-12 * np.max(np.abs(dots_ref))


def _dist_gmres_worker(rank, world, port, out_path):
    """Row-partitioned Jacobi-GMRES(m) with delayed-Gram CGS2 built from the
    parallel layer: halo exchange before every SpMM, one allreduce per phase."""
    _init(rank, world, port)
    try:
        from oracle import sylvadi_oracle as orc
        from paper_2312_02891_b200 import configs as cfgs
        from paper_2312_02891_b200.parallel import Comm, HaloPlan, RowPartition, halo_exchange
        A, _, _, _, f, _ = cfgs.build_problem("c1")
        shift, m, tol = -637.2036526571874, 20, 1e-9 * np.linalg.norm(f)
        comm = Comm()
        part = RowPartition(A.indptr, world)
        plan = HaloPlan(A, part, rank)
        op = orc.ShiftedOp(A, None, shift)
        dinv_full = orc.jacobi_dinv(op)
        dl = dinv_full[plan.r0:plan.r1]
        Al = plan.local_csr

        def apply(v):               # Op(D^-1 v) on local rows
            u = torch.from_numpy(dl * v)
            ue = halo_exchange(u[:, None], plan, comm).numpy()[:, 0]
            return Al @ ue + shift * (dl * v)

        def resid(x):
            xe = halo_exchange(torch.from_numpy(x)[:, None], plan, comm).numpy()[:, 0]
            return f[plan.r0:plan.r1, 0] - (Al @ xe + shift * x)

        def norm(v):
            return float(np.sqrt(comm.allreduce_sum(np.array([np.vdot(v, v).real]))[0]))

        b = f[plan.r0:plan.r1, 0].astype(complex)
        x = np.zeros_like(b)
        r = b.copy()
        beta = norm(r)
        it = 0
        while beta > tol:
            V = [r / beta]
            H = np.zeros((m + 1, m), complex)
            G = np.zeros((m + 1, m + 1), complex)
            cs, sn = np.zeros(m), np.zeros(m, complex)
            gv = np.zeros(m + 1, complex)
            gv[0] = beta
            k = 0
            for j in range(m):
                w = apply(V[j])
                Vm = np.array(V)
                loc = np.concatenate([Vm.conj() @ w, Vm.conj() @ V[j]])
                tot = comm.allreduce_sum(loc)            # one allreduce per phase A
                h1, gcol = tot[:j + 1], tot[j + 1:]
                G[:j + 1, j] = gcol
                G[j, :j + 1] = np.conj(gcol)
                c = h1 + (h1 - G[:j + 1, :j + 1] @ h1)
                w = w - Vm.T @ c
                hn = norm(w)                              # one allreduce per phase C
                col = np.zeros(m + 1, complex)
                col[:j + 1], col[j + 1] = c, hn
                for i in range(j):
                    a0, a1 = col[i], col[i + 1]
                    col[i] = cs[i] * a0 + sn[i] * a1
                    col[i + 1] = -np.conj(sn[i]) * a0 + cs[i] * a1
                cs[j], sn[j], rr = orc.givens(col[j], col[j + 1])
                col[j], col[j + 1] = rr, 0
                H[:, j] = col
                gv[j + 1] = -np.conj(sn[j]) * gv[j]
                gv[j] = cs[j] * gv[j]
                it += 1
                k = j + 1
                V.append(w / hn)
                if abs(gv[j + 1]) <= tol or k == m:
                    break
            y = orc._back_substitute(H[:k, :k], gv[:k])
            x = x + dl * (np.array(V[:k]).T @ y)
            r = resid(x)
            beta = norm(r)
        xs = comm.allgather(np.pad(x, (0, A.shape[0] - x.size)))
        if rank == 0:
            xg = np.concatenate([xs[q][:part.range(q)[1] - part.range(q)[0]]
                                 for q in range(world)])
            np.savez(out_path, x=xg, it=it, beta=beta)
    finally:
        dist.destroy_process_group()


def test_row_partitioned_gmres_matches_oracle(tmp_path):
    from oracle import sylvadi_oracle as orc
    from paper_2312_02891_b200 import configs as cfgs
    out = str(tmp_path / "dg.npz")
    mp.spawn(_dist_gmres_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    A, _, _, _, f, _ = cfgs.build_problem("c1")
    shift = -637.2036526571874
    op = orc.ShiftedOp(A, None, shift)
    ref = orc.gmres(op, f, 1e-9 * np.linalg.norm(f), dinv=orc.jacobi_dinv(op), restart=20,
                    orth="dcgs2")
    assert abs(int(got["it"]) - int(ref.iterations[0])) <= 2
    rel = np.linalg.norm(got["x"] - ref.solution[:, 0]) / np.linalg.norm(ref.solution[:, 0])
    assert rel < 1e-7


# -- sharded ADI: row-partitioned side groups (multigpu.ShardedAdi) -----------------------

class _GroupOracleSolver:
    """Test-side stand-in for the row-partitioned device solver: gathers the
    group's rhs slabs, solves with the oracle, returns this rank's slabs
    (counts replicated over the group, as the device solver's are)."""

    def __init__(self, side, mat, group, ranks, bounds):
        from oracle import sylvadi_oracle as orc
        self.bind = orc.Binding(side, mat, None, restart=50, orth="dcgs2")
        self.group, self.ranks, self.bounds = group, ranks, bounds
        self.me = ranks.index(dist.get_rank())

    def solve_device(self, shift, rhs, delta):
        from types import SimpleNamespace
        n = self.bounds[-1]
        pad = np.zeros((n, rhs.shape[1]), complex)
        r0, r1 = self.bounds[self.me], self.bounds[self.me + 1]
        pad[:r1 - r0] = rhs
        outs = [torch.empty((n, rhs.shape[1]), dtype=torch.complex128)
                for _ in self.ranks]
        dist.all_gather(outs, torch.from_numpy(pad), group=self.group)
        full = np.concatenate([outs[i].numpy()[:self.bounds[i + 1] - self.bounds[i]]
                               for i in range(len(self.ranks))])
        res = self.bind.solve(shift, full, delta)
        return SimpleNamespace(solution=res.solution[r0:r1].copy(),
                               residual=res.residual[r0:r1].copy(),
                               iterations=res.iterations, converged=res.converged)


class _NumpyBackend:
    def copy(self, b):
        return np.array(b, dtype=complex)

    def clone(self, b):
        return b.copy()

    def gram(self, x):
        return x.conj().T @ x

    def axpy(self, a, x, y):
        y += a * x


def _sharded_worker(rank, world, port, out_path):
    _init(rank, world, port)
    try:
        from paper_2312_02891_b200 import configs as cfgs
        from paper_2312_02891_b200.adi import AdiConfig
        from paper_2312_02891_b200.multigpu import ShardedAdi, side_groups
        from paper_2312_02891_b200.parallel import Comm, RowPartition
        from paper_2312_02891_b200.shifts import ShiftSequence
        spec = cfgs.CONFIGS["c1"]
        A, B, M, C, f, g = cfgs.build_problem("c1")
        pairs, cyclic = spec.load_shift_pairs()
        a_ranks, b_ranks = side_groups(world)
        ga = dist.new_group(a_ranks) if world > 1 else None
        gb = dist.new_group(b_ranks) if world > 1 else None
        solvers, slabs = {}, {}
        for side, mat, ranks, grp in (("A", A, a_ranks, ga), ("B", B.T.tocsr(), b_ranks, gb)):
            if rank not in ranks:
                continue
            part = RowPartition(mat.indptr, len(ranks))
            bounds = list(part.bounds)
            solvers[side] = _GroupOracleSolver(side, A if side == "A" else B, grp, ranks, bounds)
            i = ranks.index(rank)
            slabs[side] = (bounds[i], bounds[i + 1])
        cfg = AdiConfig(strategy=spec.strategy, kmax=spec.kmax)
        run = ShardedAdi(Comm(), rank, a_ranks, b_ranks, solvers, slabs, _NumpyBackend(),
                         f, g, cfg, ShiftSequence(pairs=pairs, cyclic=cyclic))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            factors, gammas, rep = run.run()
        np.savez(f"{out_path}.{rank}.npz", it_a=[r.inner_it_A for r in rep.records],
                 it_b=[r.inner_it_B for r in rep.records],
                 res=[r.scaled_res for r in rep.records], steps=rep.outer_iterations)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4])
def test_sharded_adi_matches_single_process(tmp_path, world):
    """A on ranks [0, N/2), B on [N/2, N), each side's rows split over its
    group; one all_gather of partial Grams per step: every rank reproduces the
    single-process oracle driver's steps and inner counts."""
    from oracle import sylvadi_oracle as orc
    from paper_2312_02891_b200 import configs as cfgs
    out = str(tmp_path / "sh")
    mp.spawn(_sharded_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    spec = cfgs.CONFIGS["c1"]
    A, B, M, C, f, g = cfgs.build_problem("c1")
    pairs, cyclic = spec.load_shift_pairs()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = orc.run_adi(A, B, f, g, orc.Config(strategy=spec.strategy, kmax=spec.kmax), pairs,
                          orc.Binding("A", A, None, restart=50, orth="dcgs2"),
                          orc.Binding("B", B, None, restart=50, orth="dcgs2"), cyclic=cyclic)
    for rank in range(world):
        got = np.load(f"{out}.{rank}.npz")
        assert int(got["steps"]) == ref.outer_iterations
        assert list(got["it_a"]) == [r.inner_it_A for r in ref.records]
        assert list(got["it_b"]) == [r.inner_it_B for r in ref.records]
        np.testing.assert_allclose(got["res"], [r.scaled_res for r in ref.records], rtol=1e-8)
