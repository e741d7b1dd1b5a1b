"""Loader for tests/golden/ref_precond.npz (the reference's incomplete
factorisations on seeded small operators; tests/golden/make_golden_precond.py)."""

import os

import numpy as np
import scipy.sparse as sp

from conftest import GOLD

#: case name -> (base key, mass key or None, block key)
BASES = {
    "cd12_ilu0_0": ("cd12", None, "x12"), "cd12_ilut_0.1": ("cd12", None, "x12"),
    "cd12_ilut_0.01": ("cd12", None, "x12"), "cd12_ilut_0.0001": ("cd12", None, "x12"),
    "cd24adj_ilu0_0": ("cd24", None, "x24"), "cd24adj_ilut_0.01": ("cd24", None, "x24"),
    "cd12_c_ilut": ("cd12", None, "x12"), "cd24adj_c_ilu0": ("cd24", None, "x24"),
    "lap16_ic0_0": ("lap16", None, "x16"), "lap16_ict_0.1": ("lap16", None, "x16"),
    "lap16_ict_0.01": ("lap16", None, "x16"), "pos16_ict": ("pos16", None, "x16"),
    "cd12_pencil_ilut": ("cd12", "mass12", "x12"),
    "cd12_pencil_adj_c_ilu0": ("cd12", "mass12", "x12"),
}
CASES = sorted(BASES)
LU_CASES = [c for c in CASES if "ilu" in c]
CHOL_CASES = [c for c in CASES if "ic" in c.split("_", 1)[1]]

_DATA = None


def data():
    global _DATA
    if _DATA is None:
        _DATA = dict(np.load(os.path.join(GOLD, "ref_precond.npz")))
    return _DATA


def csr(key):
    d = data()
    n = int(d[key + "_n"][0])
    return sp.csr_matrix((d[key + "_data"], d[key + "_indices"], d[key + "_indptr"]), shape=(n, n))


class Case:
    def __init__(self, name):
        d = data()
        bkey, mkey, xkey = BASES[name]
        self.name = name
        self.base = csr(bkey)
        self.mass = None if mkey is None else csr(mkey)
        self.x = d[xkey]
        self.kind = str(d[f"{name}_kind"][0])
        self.droptol = float(d[f"{name}_droptol"][0])
        self.shift = complex(d[f"{name}_shift"][0])
        self.adjoint = bool(d[f"{name}_adjoint"][0])
        self.side = "B" if self.adjoint else "A"
        self.apply = d[f"{name}_apply"]
        self.apply_spd = d.get(f"{name}_apply_spd")
        self.sign = float(d[f"{name}_sign"][0]) if f"{name}_sign" in d else 1.0
        if self.kind in ("ilu0", "ilut"):
            self.lu = tuple(d[f"{name}_{k}"] for k in ("li", "lj", "lv", "ui", "uj", "uv"))
            self.chol = None
        else:
            self.lu = None
            self.chol = tuple(d[f"{name}_{k}"] for k in ("gi", "gj", "gv"))

    def solve(self, solver):
        d = data()
        p = f"{self.name}_{solver}_"
        if p + "b" not in d:
            return None
        return {k: d[p + k] for k in ("b", "delta", "x", "iters", "norms", "conv")}
