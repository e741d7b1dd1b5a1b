"""Row-partition plans of the row-partitioned device solve (rowpart.slab_plans),
host side: the remapped slab CSR reproduces the global SpMM bit for bit, the
send/recv lists of every rank pair agree, the plan equals parallel.HaloPlan,
and a world_size-2 gloo exchange driven by the plans fills the halo rows."""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2312_02891_b200 import problems
from paper_2312_02891_b200.parallel import HaloPlan, RowPartition
from paper_2312_02891_b200.rowpart import slab_plans


def _mats():
    a2 = problems.convdiff_fd(2, 23, (lambda x, y: 10 * x, lambda x, y: 10 * y))
    a3 = problems.convdiff_fd(3, 9, (20.0, 20.0, 20.0))
    return [("2d", a2), ("3d", a3), ("3d-T", sp.csr_matrix(a3.T))]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 7])
@pytest.mark.parametrize("which", [0, 1, 2])
def test_slab_spmm_matches_global(P, which, rng):
    name, A = _mats()[which]
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    plans = slab_plans(A, P)
    assert plans[0].r0 == 0 and plans[-1].r1 == n
    x = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
    y = A @ x
    for pl in plans:
        ext = np.concatenate([x[pl.r0:pl.r1], x[pl.halo_rows]])
        yl = pl.local @ ext
        # per-row order of the global matrix is kept: identical sums
        assert np.array_equal(yl, y[pl.r0:pl.r1]), (name, P, pl.rank)
        assert pl.local.shape == (pl.n_loc, pl.n_loc + pl.n_halo)
        # local diagonal stays at local column i (Jacobi on the slab)
        d = pl.local[:, :pl.n_loc].diagonal()
        assert np.array_equal(d, A.diagonal()[pl.r0:pl.r1])


@pytest.mark.parametrize("P", [2, 3, 5])
def test_send_recv_lists_agree(P):
    _, A = _mats()[1]
    plans = slab_plans(A, P)
    for q, pq in enumerate(plans):
        assert pq.send_off[q + 1] == pq.send_off[q]          # nothing to itself
        for p, pp in enumerate(plans):
            if p == q:
                continue
            sent = pp.r0 + pp.send_rows[pp.send_off[q]:pp.send_off[q + 1]]
            got = pq.halo_rows[pq.recv_off[p]:pq.recv_off[p + 1]]
            assert np.array_equal(sent, got)


def test_plan_equals_halo_plan():
    _, A = _mats()[0]
    part = RowPartition(A.indptr, 3)
    plans = slab_plans(A, 3, part)
    for q in range(3):
        hp = HaloPlan(A, part, q)
        pl = plans[q]
        assert np.array_equal(hp.halo_rows, pl.halo_rows)
        assert (hp.local_csr != pl.local).nnz == 0
        assert np.array_equal(hp.local_csr.indices, pl.local.indices)
        for p, rows in hp.send.items():
            assert np.array_equal(rows, pl.send_rows[pl.send_off[p]:pl.send_off[p + 1]])


def test_stencil_halo_is_one_plane():
    # one neighbour plane each side for the 7-point stencil
    N = 10
    A = problems.convdiff_fd(3, N, (1.0, 1.0, 1.0))
    plans = slab_plans(A, 4)
    for pl in plans:
        nb = (pl.rank > 0) + (pl.rank < 3)
        assert pl.n_halo == nb * N * N or pl.n_halo <= 2 * N * N


# -- world_size 2 over gloo: the exchange the device path performs ---------------------

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange_worker(rank, world, port, path):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        _, A = _mats()[1]
        plans = slab_plans(A, world)
        pl = plans[rank]
        n = A.shape[0]
        x = np.arange(n * 2, dtype=np.float64).reshape(n, 2) * 0.5 + 1.0
        ext = torch.zeros((pl.n_loc + pl.n_halo, 2), dtype=torch.float64)
        ext[:pl.n_loc] = torch.from_numpy(x[pl.r0:pl.r1])
        reqs = []
        for q in range(world):
            if q == rank:
                continue
            s0, s1 = pl.send_off[q], pl.send_off[q + 1]
            if s1 > s0:
                idx = torch.from_numpy(pl.send_rows[s0:s1].astype(np.int64))
                reqs.append(dist.isend(ext[idx].contiguous(), dst=q))
            r0, r1 = pl.recv_off[q], pl.recv_off[q + 1]
            if r1 > r0:
                buf = torch.empty((r1 - r0, 2), dtype=torch.float64)
                reqs.append((dist.irecv(buf, src=q), buf, pl.n_loc + r0))
        for rq in reqs:
            if isinstance(rq, tuple):
                rq[0].wait()
                ext[rq[2]:rq[2] + rq[1].shape[0]] = rq[1]
            else:
                rq.wait()
        y = pl.local @ ext.numpy()
        ok = np.array_equal(y, (A @ x)[pl.r0:pl.r1])
        np.save(f"{path}.{rank}.npy", np.array([ok]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_halo_exchange(tmp_path):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    path = str(tmp_path / "ex")
    mp.spawn(_exchange_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    for r in range(2):
        assert bool(np.load(f"{path}.{r}.npy")[0])
