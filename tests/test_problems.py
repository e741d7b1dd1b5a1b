"""The package's problem generators reproduce the reference's bits (CPU)."""

import hashlib
import json
import os

import numpy as np
import scipy.sparse as sp

from paper_2312_02891_b200 import configs as cfgs
from paper_2312_02891_b200.problems import (convdiff_fd, fem_q1_2d, random_rhs)

from conftest import GOLD

with open(os.path.join(GOLD, "problem_hashes.json")) as fh:
    HASHES = json.load(fh)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def csr_sha(M):
    return sha(M.indptr.astype(np.int64), M.indices.astype(np.int64), M.data)


def test_config_matrices_bit_identical_to_reference():
    for name in ("c1", "c2"):
        A, B, M, C, f, g = cfgs.build_problem(name)
        ref = HASHES[name]
        assert A.nnz == ref["nnzA"] and B.nnz == ref["nnzB"]
        assert csr_sha(A) == ref["A"], name
        assert csr_sha(B) == ref["B"], name
        assert sha(f) == ref["f"] and sha(g) == ref["g"], name


def test_small_generators_bit_identical():
    assert csr_sha(convdiff_fd(3, 5, None)) == HASHES["lap3_5"]["A"]
    assert csr_sha(convdiff_fd(2, 7, (3.0, -2.0))) == HASHES["cd2_7"]["A"]


def test_stencil_known_answers():
    # test_problems.py:11-21 of the reference: 3-D diagonal -6/h^2 = -54 at n0=2? (h=1/3)
    A = convdiff_fd(3, 2, None)
    assert np.allclose(A.diagonal(), -6.0 * 9.0)
    A1 = convdiff_fd(2, 1, None)
    assert A1.toarray().tolist() == [[-16.0]]


def test_rhs_scaling():
    f, g = random_rhs(50, 30, 3, 7)
    assert abs(np.linalg.norm(f) - np.linalg.norm(g)) < 1e-12 * np.linalg.norm(f)
    f2, g2 = random_rhs(50, 30, 3, 7)
    assert np.array_equal(f, f2) and np.array_equal(g, g2)


def test_fem_pencil_structure():
    A, M = fem_q1_2d(12, (30.0, 15.0))
    n = 144
    assert A.shape == (n, n) and M.shape == (n, n)
    # 9-point pattern: interior rows have 9 entries; nnz = 9 n - 12 n0 + 4
    assert A.nnz == 9 * n - 12 * 12 + 4
    # consistent mass: symmetric positive definite, rows sum to the element area share
    Md = M.toarray()
    assert np.allclose(Md, Md.T)
    assert np.all(np.linalg.eigvalsh(Md) > 0)
    # pencil spectrum in the open left half plane
    ev = np.linalg.eigvals(np.linalg.solve(Md, A.toarray()))
    assert np.all(ev.real < 0)
    # stiffness part is symmetric, convection part skew (constant omega)
    Ad = A.toarray()
    K = -(Ad + Ad.T) / 2
    assert np.all(np.linalg.eigvalsh(K) > 0)


def test_c3_sizes():
    A, M = fem_q1_2d(1000, (30.0, 15.0))
    assert A.shape[0] == 1_000_000 and A.nnz == 8_988_004
    assert sp.isspmatrix_csr(A) and A.has_sorted_indices
