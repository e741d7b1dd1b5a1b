"""Multi-GPU layer of the inner-solve hot path.

One process per GPU, ``torch.distributed`` for the plumbing (NCCL on B200,
gloo for the CPU tests).  Two independent ways the path shards:

1. **A || B** (``SideSplitAdi``): within an outer ADI step the A- and B-system
   solves are independent once (delta_A, delta_B) are fixed (adi.py:572-576,
   SPEC.md:389).  Rank group "A" owns the A side (z_k blocks stay there), group
   "B" the B side (y_k).  The only data crossing groups per step are O(r^2)
   numbers: the six r x r Gram matrices of the fused epilogue (res, Mz / C^T y,
   w / t), from which every rank evaluates the same tolerance decision and the
   same ||w t^*||_2.

2. **Row partition** (``RowPartition``, ``HaloPlan``, ``DistributedBlocks``):
   contiguous row slabs balanced by nonzeros, a halo plan per operator (the
   remote rows the local SpMM gathers, one neighbour plane for the stencils),
   halo exchange with point-to-point send/recv, and allreduce of the per-rank
   partial sums of every block dot.  These are the communication pieces of a
   row-partitioned Krylov solve; the device kernels consume the extended
   vector [local | halo] with the column-remapped local CSR.

The scalar tolerance logic is replicated on every rank (deterministic inputs,
deterministic outputs), so no rank waits on another for a decision.
"""

import numpy as np
import scipy.sparse as sp

from .adi import (AdiConfig, SolveReport, StepRecord, Strategy, choose_tolerances, gamma,
                  tolerance_budget)
from .device import product_norm_from_grams, sigma_max_from_gram

# ---------------------------------------------------------------------------
# process-group helpers
# ---------------------------------------------------------------------------


class Comm:
    """Minimal wrapper over a torch.distributed process group."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.device = device

    def _t(self, arr):
        import torch
        t = torch.as_tensor(np.ascontiguousarray(arr))
        return t.to(self.device) if self.device is not None else t

    def allreduce_sum(self, arr):
        """Sum over ranks (fp64 / complex128 as two fp64 planes)."""
        import torch
        arr = np.asarray(arr)
        cplx = np.iscomplexobj(arr)
        base = np.stack([arr.real, arr.imag]) if cplx else arr.astype(np.float64)
        t = self._t(base)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        out = t.cpu().numpy()
        return out[0] + 1j * out[1] if cplx else out

    def allgather(self, arr):
        """List (rank order) of equally shaped arrays."""
        import torch
        t = self._t(np.asarray(arr))
        outs = [torch.empty_like(t) for _ in range(self.size)]
        self.dist.all_gather(outs, t, group=self.group)
        return [o.cpu().numpy() for o in outs]

    def broadcast(self, arr, src):
        t = self._t(np.asarray(arr))
        self.dist.broadcast(t, src=src, group=self.group)
        return t.cpu().numpy()


# ---------------------------------------------------------------------------
# row partition + halo plan
# ---------------------------------------------------------------------------


class RowPartition:
    """Contiguous row slabs with (approximately) equal nonzeros per rank."""

    def __init__(self, indptr, nranks):
        indptr = np.asarray(indptr, dtype=np.int64)
        n = indptr.size - 1
        nnz = indptr[-1]
        targets = (np.arange(1, nranks) * nnz) // nranks
        cuts = np.searchsorted(indptr, targets, side="left")
        self.bounds = np.concatenate([[0], np.clip(cuts, 0, n), [n]]).astype(np.int64)
        self.bounds = np.maximum.accumulate(self.bounds)
        self.n = n
        self.nranks = nranks

    def range(self, rank):
        return int(self.bounds[rank]), int(self.bounds[rank + 1])

    def owner(self, rows):
        return np.searchsorted(self.bounds, np.asarray(rows), side="right") - 1


class HaloPlan:
    """Local CSR (columns remapped to [local | halo]) and the send/recv lists.

    ``recv[q]`` = global rows owned by rank q that this rank's rows reference
    (sorted); ``send[q]`` = local row offsets this rank must send to rank q.
    Every rank builds every rank's recv list from the (replicated) pattern, so
    no index exchange is needed at setup.
    """

    def __init__(self, csr, part, rank):
        csr = sp.csr_matrix(csr)
        self.rank = rank
        self.part = part
        r0, r1 = part.range(rank)
        self.r0, self.r1 = r0, r1
        self.nloc = r1 - r0
        self.recv = {}
        self.send = {}
        recv_all = {q: self._needed(csr, part, q) for q in range(part.nranks)}
        mine = recv_all[rank]
        for q, rows in mine.items():
            self.recv[q] = rows
        for q in range(part.nranks):
            if q == rank:
                continue
            want = recv_all[q].get(rank)
            if want is not None and want.size:
                self.send[q] = want - r0
        # remap local columns
        halo_rows = (np.concatenate([self.recv[q] for q in sorted(self.recv)])
                     if self.recv else np.zeros(0, dtype=np.int64))
        self.halo_rows = halo_rows
        lookup = {int(g): self.nloc + i for i, g in enumerate(halo_rows)}
        blk = csr[r0:r1]
        cols = blk.indices.astype(np.int64)
        local = (cols >= r0) & (cols < r1)
        newcols = np.empty_like(cols)
        newcols[local] = cols[local] - r0
        if (~local).any():
            newcols[~local] = np.fromiter((lookup[int(c)] for c in cols[~local]),
                                          dtype=np.int64, count=int((~local).sum()))
        self.local_csr = sp.csr_matrix((blk.data, newcols, blk.indptr),
                                       shape=(self.nloc, self.nloc + halo_rows.size))
        # keep the per-row column order of the global matrix (summation order)
        self.nhalo = int(halo_rows.size)

    @staticmethod
    def _needed(csr, part, q):
        r0, r1 = part.range(q)
        cols = np.unique(csr.indices[csr.indptr[r0]:csr.indptr[r1]])
        remote = cols[(cols < r0) | (cols >= r1)]
        owners = part.owner(remote)
        return {int(o): remote[owners == o] for o in np.unique(owners)}

    @property
    def halo_bytes_per_column(self):
        return 8 * self.nhalo


def halo_exchange(x_local, plan, comm):
    """[x_local | halo] for a torch block (rows = local rows), by send/recv."""
    import torch
    reqs = []
    recv_bufs = {}
    for q in sorted(plan.recv):
        buf = torch.empty((plan.recv[q].size,) + tuple(x_local.shape[1:]),
                          dtype=x_local.dtype, device=x_local.device)
        recv_bufs[q] = buf
        reqs.append(comm.dist.irecv(buf, src=q, group=comm.group))
    for q in sorted(plan.send):
        idx = torch.as_tensor(plan.send[q], device=x_local.device)
        payload = x_local.index_select(0, idx).contiguous()
        reqs.append(comm.dist.isend(payload, dst=q, group=comm.group))
    for r in reqs:
        r.wait()
    parts = [x_local] + [recv_bufs[q] for q in sorted(plan.recv)]
    return torch.cat(parts, dim=0)


# ---------------------------------------------------------------------------
# A || B across rank groups
# ---------------------------------------------------------------------------


class SideSplitAdi:
    """ADI with the A side on rank ``a_rank`` and the B side on ``b_rank``.

    ``side_solver(shift, rhs_block, delta)`` solves this rank's side and returns
    (solution, residual, iterations, converged) as backend blocks; ``ops``
    provides ``epilogue_half(gam, mz_or_cty, res, w_or_t)`` -> the three Gram
    matrices of this side [res, Mz, w] (the per-side half of
    sad_adi_epilogue) and ``apply_mass(block)`` (M z, or C^T y; identity if
    None).  The exchange per outer step is one all_gather of 3 r x r Grams and
    the iteration counts/convergence flags.
    """

    def __init__(self, comm, side, side_solver, ops, rhs_block, config, shifts,
                 a_rank=0, b_rank=1):
        self.comm = comm
        self.side = side
        self.solve = side_solver
        self.ops = ops
        self.block = rhs_block
        self.config = config if isinstance(config, AdiConfig) else AdiConfig(**config)
        self.shifts = shifts
        self.a_rank, self.b_rank = a_rank, b_rank

    def run(self):
        cfg = self.config
        r = self.block.shape[1]
        w = self.ops.copy(self.block)
        G_own = self.ops.gram(w)
        G_all = self.comm.allgather(G_own)
        Gw, Gt = G_all[self.a_rank], G_all[self.b_rank]
        res0 = product_norm_from_grams(Gw, Gt)
        rep = SolveReport(rhs_norm=res0, strategy=cfg.strategy)
        factors, gammas = [], []
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
            if self.side == "A":
                sol, resid, its, conv = self.solve(beta, w, dec.delta_A if dec.delta_A > 0 else 1.0)
                g_side = gam
            else:
                sol, resid, its, conv = self.solve(alpha, w, dec.delta_B if dec.delta_B > 0 else 1.0)
                g_side = np.conj(gam)
            mass = self.ops.apply_mass(sol)
            Gr, Gm, Gn = self.ops.epilogue_half(g_side, mass, resid, w)
            meta = np.array([float(np.sum(its)), float(np.all(conv))])
            packed = np.concatenate([np.stack([Gr, Gm, Gn]).ravel().view(np.float64), meta])
            got = self.comm.allgather(packed)
            unpack = []
            for arr in got:
                g3 = arr[:-2].view(np.complex128).reshape(3, r, r)
                unpack.append((g3, arr[-2:]))
            (GrA, GmA, GwA), metaA = unpack[self.a_rank]
            (GrB, GmB, GtB), metaB = unpack[self.b_rank]
            rA, rB = sigma_max_from_gram(GrA), sigma_max_from_gram(GrB)
            u += abs(gam) * sigma_max_from_gram(GmA) * rB
            v += abs(gam) * sigma_max_from_gram(GmB) * rA
            Gw, Gt = GwA, GtB
            res = product_norm_from_grams(Gw, Gt)
            factors.append(sol)
            gammas.append(gam)
            k_done = k
            rep.records.append(StepRecord(
                step=k, scaled_res=res / res0, delta_A=dec.delta_A, delta_B=dec.delta_B,
                achieved_rA=rA, achieved_rB=rB, inner_it_A=int(metaA[0]),
                inner_it_B=int(metaB[0]), u=u, v=v, wall_ms=0.0,
                a_converged=bool(metaA[1]), b_converged=bool(metaB[1]),
                clamped_A_min=dec.clamped_A_min, clamped_B_min=dec.clamped_B_min))
            if res < cfg.outer_tolerance * res0:
                break
        rep.converged = bool(res < cfg.outer_tolerance * res0)
        rep.outer_iterations = k_done
        rep.final_scaled_residual = res / res0
        return factors, gammas, rep


class DeviceSideOps:
    """SideSplitAdi ops on the device (libsylvadi_b200 kernels)."""

    def __init__(self, mass=None, transpose=False, device=0):
        self.mass = mass
        self.transpose = transpose
        self.device = device

    def copy(self, block):
        import torch
        t = torch.as_tensor(block)
        return t.to(torch.device("cuda", self.device)).clone()

    def gram(self, x):
        from .device import gram
        return gram(x, device=self.device)

    def apply_mass(self, x):
        if self.mass is None:
            return x
        return self.mass.apply(x, transpose=self.transpose)

    def epilogue_half(self, gam, mz, res, w):
        from .device import axpy, gram
        axpy(gam, mz, w, device=self.device)
        return gram(res, device=self.device), gram(mz, device=self.device), \
            gram(w, device=self.device)
