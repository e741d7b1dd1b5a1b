"""Sharded ADI across processes: one process per GPU.

The A side is row-partitioned over the ranks ``a_ranks`` and the B side over
``b_ranks`` (disjoint groups on N >= 2 GPUs: A on the first half, B on the
second, BASELINE config 5; one process may own both sides on one GPU).  Per
outer step (adi.py:510-537, run_with_state adi.py:553-607):

* each group solves its side on its row slabs (``rowpart.RowPartitionedGmres``
  with an NCCL communicator over the group: halo exchange + all-reduce inside
  the Krylov loop, nothing else crosses GPUs inside a solve);
* each rank updates its slab of w (or t) and forms its LOCAL partial Gram
  matrices of the inner residual, of z (or y) and of the updated w (or t);
* ONE all-gather over the world carries every rank's partials (3 r x r per
  owned side) and the side's iteration counts; every rank sums the partials of
  each group in rank order, so every rank evaluates the same ||res||,
  ||w t^*||, u, v and the same next tolerance decision (adi.py:347-408) --
  the exchange per step is O(N r^2), independent of n.

The factors Z, Y stay distributed (row slabs on their owners).
"""

import numpy as np

from .adi import (AdiConfig, SolveReport, StepRecord, choose_tolerances, gamma,
                  tolerance_budget)
from .device import product_norm_from_grams, sigma_max_from_gram


def side_groups(world):
    """(a_ranks, b_ranks): disjoint halves for N >= 2, both sides on rank 0 for N = 1."""
    if world == 1:
        return [0], [0]
    h = world // 2
    return list(range(h)), list(range(h, world))


class ShardedAdi:
    """ADI with row-partitioned sides on rank groups.

    ``solvers[side]`` (only for the sides this rank owns) has
    ``solve_device(shift, rhs_slab, delta)`` returning an object with
    ``solution``, ``residual``, ``iterations``, ``converged`` (slabs; counts
    replicated over the group).  ``backend`` provides ``copy(host_slab)``,
    ``gram(x)`` (local partial X^H X, numpy r x r), ``axpy(a, x, y)`` (y += a x,
    in place).  ``comm`` is ``parallel.Comm`` over the world (all_gather).
    ``slabs[side] = (r0, r1)`` are this rank's rows of each owned side.
    """

    def __init__(self, comm, rank, a_ranks, b_ranks, solvers, slabs, backend, f, g, config,
                 shifts):
        self.comm, self.rank = comm, rank
        self.a_ranks, self.b_ranks = list(a_ranks), list(b_ranks)
        self.solvers, self.slabs, self.be = solvers, slabs, backend
        self.config = config if isinstance(config, AdiConfig) else AdiConfig(**config)
        self.shifts = shifts
        self.r = f.shape[1]
        self.mine = [s for s, ranks in (("A", self.a_ranks), ("B", self.b_ranks)) if rank in ranks]
        self.rhs = {}                       # this rank's slabs of f and g (device)
        for side in self.mine:
            r0, r1 = slabs[side]
            src = f if side == "A" else g
            self.rhs[side] = backend.copy(src[r0:r1])
        self.blocks = {}

    # packed per-rank message: for side A then B: [res, z, w] Grams (3 r^2
    # complex) + [sum of iterations, all converged]; zeros for sides not owned
    def _pack(self, grams, meta):
        r = self.r
        out = []
        for side in ("A", "B"):
            g3 = grams.get(side, np.zeros((3, r, r), complex))
            out.append(np.asarray(g3, complex).ravel().view(np.float64))
            out.append(np.asarray(meta.get(side, (0.0, 1.0)), np.float64))
        return np.concatenate(out)

    def _unpack(self, arrs):
        r = self.r
        n3 = 3 * r * r * 2
        sums, metas = {}, {}
        for side, ranks, base in (("A", self.a_ranks, 0), ("B", self.b_ranks, n3 + 2)):
            tot = np.zeros((3, r, r), complex)
            for q in ranks:                      # rank order: identical on every rank
                tot = tot + arrs[q][base:base + n3].view(np.complex128).reshape(3, r, r)
            sums[side] = tot
            metas[side] = arrs[ranks[0]][base + n3:base + n3 + 2]
        return sums, metas

    def _exchange(self, grams, meta):
        return self._unpack(self.comm.allgather(self._pack(grams, meta)))

    def run(self):
        cfg = self.config
        be = self.be
        self.blocks = {s: be.clone(self.rhs[s]) for s in self.mine}   # w, t start at f, g
        # initial ||f g^*||: Grams of the local slabs of f and g
        g0 = {s: np.stack([np.zeros((self.r, self.r), complex)] * 2 + [be.gram(self.blocks[s])])
              for s in self.mine}
        sums, _ = self._exchange(g0, {})
        Gw, Gt = sums["A"][2], sums["B"][2]
        res0 = product_norm_from_grams(Gw, Gt)
        rep = SolveReport(rhs_norm=res0, strategy=cfg.strategy)
        factors = {s: [] for s in self.mine}
        gammas = []
        u = v = 0.0
        gap = cfg.gap_budget if cfg.gap_budget is not None else cfg.outer_tolerance * res0
        res = res0
        k_done = 0
        for k in range(1, cfg.kmax + 1):
            eps_hat = tolerance_budget(cfg, k, u, v, gap)
            dec = choose_tolerances(cfg, k, sigma_max_from_gram(Gw), sigma_max_from_gram(Gt),
                                    eps_hat)
            alpha, beta = (complex(s) for s in self.shifts.at(k))
            gam = gamma(alpha, beta)
            grams, meta = {}, {}
            for side in self.mine:
                if side == "A":
                    shift, delta, gs = beta, dec.delta_A, gam
                else:
                    shift, delta, gs = alpha, dec.delta_B, np.conj(gam)
                solver = self.solvers[side]
                out = solver.solve_device(shift, self.blocks[side], delta if delta > 0 else 1.0)
                # M z (A side) or C^T y (B side); identity mass when None
                mass = getattr(solver, "mass", None)
                mz = out.solution if mass is None else mass.apply(out.solution,
                                                                  transpose=(side == "B"))
                be.axpy(gs, mz, self.blocks[side])
                grams[side] = np.stack([be.gram(out.residual), be.gram(mz),
                                        be.gram(self.blocks[side])])
                meta[side] = (float(np.sum(out.iterations)), float(np.all(out.converged)))
                factors[side].append(out.solution)
            sums, metas = self._exchange(grams, meta)
            GrA, GzA, GwA = sums["A"]
            GrB, GyB, GtB = sums["B"]
            rA, rB = sigma_max_from_gram(GrA), sigma_max_from_gram(GrB)
            u += abs(gam) * sigma_max_from_gram(GzA) * rB
            v += abs(gam) * sigma_max_from_gram(GyB) * rA
            Gw, Gt = GwA, GtB
            res = product_norm_from_grams(Gw, Gt)
            gammas.append(gam)
            k_done = k
            rep.records.append(StepRecord(
                step=k, scaled_res=res / res0, delta_A=dec.delta_A, delta_B=dec.delta_B,
                achieved_rA=rA, achieved_rB=rB, inner_it_A=int(metas["A"][0]),
                inner_it_B=int(metas["B"][0]), u=u, v=v, wall_ms=0.0,
                a_converged=bool(metas["A"][1]), b_converged=bool(metas["B"][1]),
                clamped_A_min=dec.clamped_A_min, clamped_B_min=dec.clamped_B_min))
            if res < cfg.outer_tolerance * res0:
                break
        rep.converged = bool(res < cfg.outer_tolerance * res0)
        rep.outer_iterations = k_done
        rep.final_scaled_residual = res / res0
        return factors, gammas, rep


class DeviceBackend:
    """ShardedAdi block ops on this rank's device (libsylvadi_b200 kernels)."""

    def __init__(self, device=0, dtype=None):
        self.device = device
        self.dtype = dtype

    def copy(self, host):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(host))
        if self.dtype is not None:
            t = t.to(self.dtype)
        return t.to(torch.device("cuda", self.device)).contiguous()

    def clone(self, x):
        return x.clone()

    def gram(self, x):
        from .device import gram
        return gram(x, device=self.device)

    def axpy(self, a, x, y):
        from .device import axpy
        axpy(a, x, y, device=self.device)


def make_sharded(problem, config, shifts, *, restart=30, flexible=False, device=None,
                 force_rowpart=False):
    """One process per GPU (torch.distributed initialised, any backend): build
    this rank's side solvers and the ShardedAdi driver: a side owned by a
    group of several ranks is row-partitioned (NCCL communicator over the
    group); a side on one GPU uses the persistent engine unless
    ``force_rowpart``."""
    import torch
    import torch.distributed as dist
    from .krylov import GpuGmresBinding
    from .parallel import Comm
    from .rowpart import RowPartitionedGmres
    world = dist.get_world_size()
    rank = dist.get_rank()
    dev = rank % max(1, torch.cuda.device_count()) if device is None else device
    torch.cuda.set_device(dev)
    a_ranks, b_ranks = side_groups(world)
    # every rank creates both subgroups, in the same order
    ga = dist.new_group(a_ranks) if world > 1 else None
    gb = dist.new_group(b_ranks) if world > 1 else None
    pairs = [shifts.at(k) for k in range(1, config.kmax + 1)]
    cplx = any(complex(a).imag or complex(b).imag for a, b in pairs)
    tdtype = torch.complex128 if cplx else torch.float64
    kw = dict(max_iterations=config.max_inner_iterations, restart=restart, flexible=flexible,
              device=dev)
    solvers, slabs = {}, {}
    for side, ranks, grp in (("A", a_ranks, ga), ("B", b_ranks, gb)):
        if rank not in ranks:
            continue
        base, mass = (problem.A, problem.M) if side == "A" else (problem.B, problem.C)
        kind = config.precond_kind_A if side == "A" else config.precond_kind_B
        from .adi import AUTO_RING_BLOCK_BYTES
        big = ((problem.n if side == "A" else problem.m) * problem.r * 16 >= AUTO_RING_BLOCK_BYTES
               and problem.r <= 8)
        if len(ranks) == 1 and big and not force_rowpart:
            # a large side on one GPU: the ring multi-kernel engine on one slab
            # (DeviceAdi's engine="auto" rule; config 5 at 2 GPUs)
            s = RowPartitionedGmres(side, base, mass, "iterative", kind, nranks=1, comm="local",
                                    **kw)
            solvers[side] = s
            slabs[side] = (0, s.n)
        elif len(ranks) == 1 and not force_rowpart:
            # a side on one GPU: the persistent single-GPU engine (also takes a
            # mass matrix, config 3 at 2 GPUs = A || B)
            s = GpuGmresBinding(side, base, mass, "iterative", kind, engine="persistent", **kw)
            solvers[side] = s
            slabs[side] = (0, s.n)
        else:
            s = RowPartitionedGmres(side, base, mass, "iterative", kind, nranks=len(ranks),
                                    group=grp, comm="nccl", **kw)
            solvers[side] = s
            slabs[side] = (s.plans[0].r0, s.plans[0].r1)
    comm_dev = torch.device("cuda", dev) if dist.get_backend() == "nccl" else None
    return ShardedAdi(Comm(device=comm_dev), rank, a_ranks, b_ranks, solvers, slabs,
                      DeviceBackend(dev, tdtype), problem.f, problem.g, config, shifts)
