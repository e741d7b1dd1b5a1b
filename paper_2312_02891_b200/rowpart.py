"""Row-partitioned inner solves.

One shifted operator is split into contiguous row slabs balanced by nonzeros
(``parallel.RowPartition``); each rank owns a slab, the rows of the Krylov
blocks that belong to it, and a halo plan (the remote rows its SpMM gathers).
The solve is ``sad_dist_gmres_solve``: the multi-kernel engine's step sequence
on every rank, halo exchange before each SpMM, every block dot all-reduced
before its (replicated) finisher -- delayed-Gram CGS2 by default (two basis
sweeps, two all-reduces per step; ``orth="cgs2"``: four and three).  Same
contract as the single-GPU engine
(SURVEY 8a items 1-6); reductions are summed per rank then over ranks, so the
results agree with one GPU to rounding, not bit for bit.

``RowPartitionedGmres`` has ``GpuGmresBinding``'s constructor shape and
``solve`` / ``solve_device`` (adi.py:422-488, krylov.py:41-70), plus:

* ``nranks`` -- number of slabs;
* ``comm="local"`` -- all ranks in this process on one device, kernels issued
  in rank order, the all-reduce a device sum and send/recv device copies (no
  kernel waits for another rank; the one-GPU test vehicle, B200_PROFILING.md);
* ``comm="nccl"`` -- one process per GPU: this process is rank
  ``torch.distributed.get_rank(group)`` of the ``nranks`` ranks, the NCCL
  communicator is created by the library from a unique id broadcast over
  ``group``; ``solve_device`` takes and returns this rank's slab.

The B side solves with ``B^T + conj(sigma) I``: the slab plan is built on the
explicit transpose (same per-row summation order as the library's adjoint,
sad_capi.cu host_transpose) and the shift is conjugated.  A non-identity mass
(config 3) is not row-partitioned (BASELINE.json runs it A || B).
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .device import as_csr, current_stream_handle
from .krylov import InnerSolveResult, validate_request
from .parallel import RowPartition

_KIND = {"none": _lib.SAD_PRECOND_NONE, "jacobi": _lib.SAD_PRECOND_JACOBI}


@dataclass
class SlabPlan:
    """One rank's slab: rows [r0, r1), the remapped local CSR (columns
    [local | halo], the global matrix's per-row order), halo rows grouped by
    owner (recv_off), and the local rows each peer needs (send_off/send_rows)."""
    rank: int
    r0: int
    r1: int
    local: sp.csr_matrix
    halo_rows: np.ndarray
    recv_off: np.ndarray
    send_off: np.ndarray
    send_rows: np.ndarray

    @property
    def n_loc(self):
        return self.r1 - self.r0

    @property
    def n_halo(self):
        return int(self.halo_rows.size)


def slab_plans(mat, nranks, part=None):
    """Slab plans of every rank (vectorised; the same plan as parallel.HaloPlan)."""
    csr = as_csr(mat)
    n = csr.shape[0]
    if csr.shape[1] != n:
        raise ValueError("row partitioning needs a square operator")
    part = part or RowPartition(csr.indptr, nranks)
    P = part.nranks
    halos, locals_ = [], []
    for q in range(P):
        r0, r1 = part.range(q)
        lo, hi = csr.indptr[r0], csr.indptr[r1]
        cols = csr.indices[lo:hi].astype(np.int64)
        remote = (cols < r0) | (cols >= r1)
        halo = np.unique(cols[remote])                 # sorted => grouped by owner
        newcols = cols - r0
        newcols[remote] = (r1 - r0) + np.searchsorted(halo, cols[remote])
        indptr = (csr.indptr[r0:r1 + 1] - lo).astype(np.int64)
        locals_.append(sp.csr_matrix((csr.data[lo:hi], newcols, indptr),
                                     shape=(r1 - r0, r1 - r0 + halo.size)))
        halos.append(halo)
    plans = []
    for q in range(P):
        r0, r1 = part.range(q)
        own = part.owner(halos[q]) if halos[q].size else np.zeros(0, dtype=np.int64)
        recv_off = np.zeros(P + 1, dtype=np.int64)
        recv_off[1:] = np.cumsum(np.bincount(own, minlength=P))
        send_off = np.zeros(P + 1, dtype=np.int64)
        send = []
        for p in range(P):
            if p != q and halos[p].size:
                want = halos[p][(halos[p] >= r0) & (halos[p] < r1)] - r0
            else:
                want = np.zeros(0, dtype=np.int64)
            send.append(want)
            send_off[p + 1] = send_off[p] + want.size
        send_rows = (np.concatenate(send) if send else np.zeros(0)).astype(np.int32)
        plans.append(SlabPlan(q, r0, r1, locals_[q], halos[q], recv_off, send_off, send_rows))
    return plans


def _ptrs(vals):
    arr = (ctypes.c_void_p * len(vals))(*[ctypes.c_void_p(v) if not isinstance(v, ctypes.c_void_p)
                                          else v for v in vals])
    return arr


class _Handle:
    def __init__(self, h, destroy):
        self.h, self._destroy = h, destroy

    def __del__(self):
        if self.h:
            try:
                getattr(_lib.load(), self._destroy)(self.h)
            except Exception:
                pass
            self.h = None


class _Comm:
    """sad_comm: an in-process group of ``nranks`` ranks, or NCCL."""

    def __init__(self, ctx, nranks, kind="local", group=None):
        lib = _lib.load()
        h = ctypes.c_void_p()
        self.kind = kind
        if kind == "local":
            _lib.check(lib.sad_comm_create_local(ctx, nranks, ctypes.byref(h)), ctx)
            self.rank = None
        elif kind == "nccl":
            import torch.distributed as dist
            self.rank = dist.get_rank(group)
            if dist.get_world_size(group) != nranks:
                raise ValueError("nranks must equal the process group size")
            uid = (ctypes.c_uint8 * 128)()
            if self.rank == 0:
                rc = lib.sad_comm_unique_id(uid)
                if rc != _lib.SAD_OK:
                    raise _lib.DeviceError("NCCL unavailable: " +
                                           lib.sad_comm_nccl_error().decode())
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0)
                                       if group is not None else 0, group=group)
            uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
            _lib.check(lib.sad_comm_create_nccl(ctx, nranks, self.rank, uid, ctypes.byref(h)), ctx)
        else:
            raise ValueError("comm must be 'local' or 'nccl'")
        self.handle = _Handle(h, "sad_comm_destroy")
        self.nranks = nranks

    @property
    def h(self):
        return self.handle.h


class _OpRef:
    """A single-GPU DeviceOperator standing in for the one slab of a P = 1 group."""

    def __init__(self, dop):
        self.dop = dop

    @property
    def h(self):
        return self.dop.handle


class RowPartitionedGmres:
    """Jacobi-GMRES(m)/FGMRES(m) on a row-partitioned operator (see module doc)."""

    def __init__(self, side, base, mass=None, mode="iterative", precond_kind="jacobi",
                 droptol=0.1, max_iterations=1000, *, nranks=2, restart=50, flexible=False,
                 device=0, comm="local", group=None, orth="dcgs2"):
        if side not in ("A", "B"):
            raise ValueError("side must be 'A' or 'B'")
        if mode != "iterative":
            raise NotImplementedError("direct inner solves are outside the GPU hot path")
        if precond_kind not in _KIND:
            raise ValueError(f"preconditioner {precond_kind!r} is not available on the GPU path")
        if mass is not None and int(nranks) != 1:
            raise NotImplementedError("a non-identity mass matrix is not row-partitioned "
                                      "(generalised pencils run A || B, BASELINE config 3)")
        if orth not in ("dcgs2", "cgs2"):
            raise ValueError("orth must be 'dcgs2' or 'cgs2'")
        self.orth = orth
        self.side, self.mode, self.precond_kind = side, mode, precond_kind
        self.droptol = droptol
        self.max_iterations = int(max_iterations)
        self.restart, self.flexible = int(restart), bool(flexible)
        self.device = device
        self.mass = None
        self._ctx = _lib.context(device)
        self._base_dm = None
        if mass is not None:
            # one slab: the whole generalised pencil, assembled per shift by the
            # single-GPU operator (sad_op_create); DeviceAdi reads .mass for M z / C^T y
            from .device import DeviceMatrix
            adj = (side == "B")
            self._base_dm = base if isinstance(base, DeviceMatrix) else DeviceMatrix(base, adj, device)
            self.mass = mass if isinstance(mass, DeviceMatrix) else DeviceMatrix(mass, adj, device)
        csr = as_csr(base)
        if side == "B":
            csr = as_csr(csr.T.tocsr())
        self.n = csr.shape[0]
        self.nranks = int(nranks)
        self.comm = _Comm(self._ctx, self.nranks, comm, group)
        plans = slab_plans(csr, self.nranks)
        self.all_plans = plans
        self.plans = plans if comm == "local" else [plans[self.comm.rank]]
        lib = _lib.load()
        self._slabs, self._halos = [], []
        for pl in self.plans:
            loc = pl.local
            rp = np.ascontiguousarray(loc.indptr, dtype=np.int32)
            ci = np.ascontiguousarray(loc.indices, dtype=np.int32)
            va = np.ascontiguousarray(loc.data, dtype=np.float64)
            h = ctypes.c_void_p()
            _lib.check(lib.sad_local_csr_create(self._ctx, loc.shape[0], loc.shape[1], loc.nnz,
                                                rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
                                                ctypes.byref(h)), self._ctx)
            self._slabs.append(_Handle(h, "sad_csr_destroy"))
            so = np.ascontiguousarray(pl.send_off, dtype=np.int64)
            sr = np.ascontiguousarray(pl.send_rows, dtype=np.int32)
            ro = np.ascontiguousarray(pl.recv_off, dtype=np.int64)
            hh = ctypes.c_void_p()
            _lib.check(lib.sad_halo_create(self._ctx, self.nranks, pl.rank, pl.n_loc, pl.n_halo,
                                           so.ctypes.data, sr.ctypes.data if sr.size else None,
                                           ro.ctypes.data, ctypes.byref(hh)), self._ctx)
            self._halos.append(_Handle(hh, "sad_halo_destroy"))
        self._ops = {}
        self._ws = {}

    @property
    def nl(self):
        return len(self.plans)

    def halo_bytes_per_column(self, dtype_bytes=8):
        return sum(pl.n_halo for pl in self.all_plans) * dtype_bytes

    # -- caches -------------------------------------------------------------
    def operator(self, shift):
        """Per-rank slab operators for ``shift`` (B side: conj(shift) on B^T)."""
        shift = complex(shift)
        ops = self._ops.get(shift)
        if ops is None:
            s = np.conj(shift) if self.side == "B" else shift
            lib = _lib.load()
            ops = []
            if self.mass is not None:
                from .device import DeviceOperator
                dop = DeviceOperator(self._base_dm, self.mass, shift, adjoint=(self.side == "B"),
                                     precond_kind=self.precond_kind)
                ops.append(_OpRef(dop))
            else:
                for slab in self._slabs:
                    h = ctypes.c_void_p()
                    _lib.check(lib.sad_local_op_create(self._ctx, slab.h, s.real, s.imag,
                                                       _KIND[self.precond_kind], ctypes.byref(h)),
                               self._ctx)
                    ops.append(_Handle(h, "sad_op_destroy"))
            import torch
            stream = torch.cuda.current_stream(torch.device("cuda", self.device))
            _lib.check(lib.sad_dist_op_setup(self.comm.h, self.nl, _ptrs([o.h for o in ops]),
                                             _ptrs([hh.h for hh in self._halos]),
                                             current_stream_handle(stream)), self._ctx)
            self._ops[shift] = ops
        return ops

    def workspaces(self, r, dtype):
        key = (r, dtype)
        ws = self._ws.get(key)
        if ws is None:
            lib = _lib.load()
            ws = []
            for pl in self.plans:
                h = ctypes.c_void_p()
                _lib.check(lib.sad_dist_gmres_create(self._ctx, pl.n_loc, pl.n_loc + pl.n_halo, r,
                                                     dtype, self.restart,
                                                     1 if self.flexible else 0,
                                                     ctypes.byref(h)), self._ctx)
                ws.append(_Handle(h, "sad_gmres_destroy"))
                _lib.check(lib.sad_gmres_set_option(h, _lib.SAD_OPT_DIST_ORTH,
                                                    1 if self.orth == "dcgs2" else 0), self._ctx)
            self._ws[key] = ws
        return ws

    # -- solves -------------------------------------------------------------
    def _slab_views(self, block):
        """Row slabs of this process's ranks: views of a full (n, r) block
        (local group), or the block itself (NCCL: it is this rank's slab)."""
        if self.comm.kind == "local":
            return [block[pl.r0:pl.r1] for pl in self.plans]
        return [block]

    def solve_device(self, shift, rhs, delta, x=None, res=None, stream=None):
        """Device solve.  Local group: rhs/x/res are full (n, r) torch blocks
        (ranks work on their row slabs in place).  NCCL: this rank's slab."""
        import torch
        from .krylov import DeviceSolveResult
        if delta <= 0.0:
            raise ValueError("abs_tolerance must be positive")
        rows, r = rhs.shape
        want = self.n if self.comm.kind == "local" else self.plans[0].n_loc
        if rows != want:
            raise ValueError("rhs rows do not match the operator (slab) size")
        if r > 8:
            raise ValueError("row-partitioned solves take at most 8 columns")
        ops = self.operator(shift)
        complex_shift = complex(shift).imag != 0.0
        if rhs.dtype == torch.float64 and complex_shift:
            raise ValueError("complex shift requires a complex128 block")
        dtype = _lib.SAD_F64 if rhs.dtype == torch.float64 else _lib.SAD_C128
        x = torch.empty_like(rhs) if x is None else x
        res = torch.empty_like(rhs) if res is None else res
        ws = self.workspaces(r, dtype)
        b_s, x_s, r_s = self._slab_views(rhs), self._slab_views(x), self._slab_views(res)
        for t in b_s + x_s + r_s:
            if not t.is_contiguous():
                raise ValueError("blocks must be row-major contiguous")
        iters = np.zeros(r, dtype=np.int64)
        norms = np.zeros(r, dtype=np.float64)
        conv = np.zeros(r, dtype=np.uint8)
        rc = _lib.load().sad_dist_gmres_solve(
            self.comm.h, self.nl, _ptrs([w.h for w in ws]), _ptrs([o.h for o in ops]),
            _ptrs([hh.h for hh in self._halos]), _ptrs([t.data_ptr() for t in b_s]),
            _ptrs([t.data_ptr() for t in x_s]), _ptrs([t.data_ptr() for t in r_s]),
            float(delta) / r, self.max_iterations, current_stream_handle(stream),
            iters.ctypes.data, norms.ctypes.data, conv.ctypes.data)
        _lib.check(rc, self._ctx)
        return DeviceSolveResult(solution=x, residual=res, achieved_residual_norms=norms,
                                 iterations=iters, converged=conv.astype(bool))

    def apply_device(self, shift, x):
        """y = Op x through the slab operators and one halo exchange (full
        block for the local group, this rank's slab for NCCL)."""
        import torch
        ops = self.operator(shift)
        dtype = _lib.SAD_F64 if x.dtype == torch.float64 else _lib.SAD_C128
        r = x.shape[1]
        xs = self._slab_views(x)
        ext = [torch.zeros((pl.n_loc + pl.n_halo, r), dtype=x.dtype, device=x.device)
               for pl in self.plans]
        for e, s in zip(ext, xs):
            e[:s.shape[0]] = s
        y = torch.empty_like(x)
        ys = self._slab_views(y)
        rc = _lib.load().sad_dist_op_apply(
            self.comm.h, self.nl, _ptrs([o.h for o in ops]), _ptrs([hh.h for hh in self._halos]),
            r, dtype, _ptrs([e.data_ptr() for e in ext]), _ptrs([t.data_ptr() for t in ys]),
            current_stream_handle())
        _lib.check(rc, self._ctx)
        return y

    def allreduce_(self, tensors):
        """In-place sum over ranks of float64/complex128 device tensors (one per
        local rank)."""
        import torch
        bufs = [torch.view_as_real(t) if t.is_complex() else t for t in tensors]
        rc = _lib.load().sad_dist_allreduce(self.comm.h, self.nl, _ptrs([b.data_ptr() for b in bufs]),
                                            bufs[0].numel(), current_stream_handle())
        _lib.check(rc, self._ctx)
        return tensors

    def solve(self, shift, rhs, delta):
        """SolverBinding.solve (adi.py:473-488) on host numpy blocks (local
        group: the whole operator; NCCL: this rank's slab)."""
        import torch
        want = self.n if self.comm.kind == "local" else self.plans[0].n_loc
        rhs = validate_request(want, rhs, delta)
        real = complex(shift).imag == 0.0 and not np.any(rhs.imag)
        dev = torch.device("cuda", self.device)
        b = torch.from_numpy(np.ascontiguousarray(rhs.real if real else rhs)).to(dev)
        out = self.solve_device(shift, b, delta)
        torch.cuda.current_stream(dev).synchronize()
        sol = out.solution.cpu().numpy().astype(np.complex128)
        res = out.residual.cpu().numpy().astype(np.complex128)
        return InnerSolveResult(solution=sol, residual=res,
                                achieved_residual_norms=out.achieved_residual_norms,
                                iterations=out.iterations, converged=out.converged)
