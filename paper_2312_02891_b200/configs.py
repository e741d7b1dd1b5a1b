"""The BASELINE.json configurations, with the pins SURVEY.md section 8d asks for.

Each entry builds the seeded problem exactly as the reference would
(``problems.py`` generators, Philox seed) and names the pinned shift file
(``configs/shifts_<name>.json``, produced once by the reference's own
``pencil_ritz_sets`` + ``heuristic_shifts`` in the build container by
``tests/golden/make_golden.py``), the outer-step cap kmax and the inner
GMRES restart length.
"""

import json
import os
from dataclasses import dataclass, field

import numpy as np

from .problems import convdiff_fd, fem_q1_2d, random_rhs

_HERE = os.path.dirname(os.path.abspath(__file__))
SHIFT_DIR = os.path.join(os.path.dirname(_HERE), "configs")


@dataclass
class ConfigSpec:
    name: str
    description: str
    r: int
    seed: int
    kmax: int
    restart: int
    flexible: bool
    npairs: int
    outer_tolerance: float = 1e-8
    strategy: str = "dynamic_mid_bl"
    extra: dict = field(default_factory=dict)

    @property
    def shift_file(self):
        return os.path.join(SHIFT_DIR, f"shifts_{self.extra.get('shifts', self.name)}.json")

    def load_shift_pairs(self):
        """ShiftSequence JSON (shifts.py:53-67 layout) -> list of (alpha, beta)."""
        with open(self.shift_file) as fh:
            payload = json.load(fh)
        pairs = [(complex(a[0], a[1]), complex(b[0], b[1]))
                 for a, b in payload["pairs"]]
        return pairs, bool(payload.get("cyclic", True))


def _c1_matrices():
    A = convdiff_fd(2, 64, (lambda x, y: 10.0 * x, lambda x, y: 10.0 * y))
    B = convdiff_fd(2, 48, (lambda x, y: 50.0 * y, lambda x, y: -50.0 * x))
    return A, B, None, None


def _c2_matrices():
    A = convdiff_fd(3, 40, (20.0, 20.0, 20.0))
    B = convdiff_fd(3, 30, (lambda x, y, z: 5.0 * x, lambda x, y, z: -5.0 * y,
                            lambda x, y, z: 5.0 * z))
    return A, B, None, None


def _c3_matrices(n0_a=1000, n0_b=700):
    A, M = fem_q1_2d(n0_a, (30.0, 15.0))
    B, C = fem_q1_2d(n0_b, (0.0, 10.0))
    return A, B, M, C


def _c4_matrix(n0=4096):
    return convdiff_fd(2, n0, (100.0, 100.0))


def _c5_matrices(n0_a=200, n0_b=160):
    A = convdiff_fd(3, n0_a, (lambda x, y, z: 50.0 * x, lambda x, y, z: 50.0 * y,
                              lambda x, y, z: 50.0 * z))
    B = convdiff_fd(3, n0_b, (10.0, -10.0, 10.0))
    return A, B, None, None


def _c3s_matrices():
    """Config 3 at reduced size (same generator, operators and convection)."""
    return _c3_matrices(n0_a=48, n0_b=40)


def _c3m_matrices():
    """Config 3 at an intermediate size (250^2 / 175^2) with the FULL-size
    problem's pinned shifts: the regime where the small pair alpha ~ -1535,
    beta ~ -1575 makes the A-side Jacobi-GMRES(40) stagnate."""
    return _c3_matrices(n0_a=250, n0_b=175)


def _c5s_matrices():
    """Config 5 operator family at proxy size (n0=16 / 13)."""
    return _c5_matrices(n0_a=16, n0_b=13)


CONFIGS = {
    "c1": ConfigSpec("c1", "2-D conv-diff 64^2 / 48^2, r=1, GMRES(50)",
                     r=1, seed=0, kmax=150, restart=50, flexible=False,
                     npairs=10),
    "c2": ConfigSpec("c2", "3-D conv-diff 40^3 / 30^3, r=2, complex, FGMRES(30)",
                     r=2, seed=0, kmax=150, restart=30, flexible=True,
                     npairs=12),
    "c3": ConfigSpec("c3", "2-D Q1 FEM pencils 1000^2 / 700^2, r=3, GMRES(40)",
                     r=3, seed=0, kmax=200, restart=40, flexible=False,
                     npairs=10),
    "c4": ConfigSpec("c4", "inner-solve microbenchmark 4096^2, r=8, 100 GMRES its",
                     r=8, seed=0, kmax=1, restart=100, flexible=False,
                     npairs=0),
    "c5": ConfigSpec("c5", "3-D conv-diff 200^3 / 160^3, r=4, GMRES(30)",
                     r=4, seed=0, kmax=700, restart=30, flexible=False,
                     npairs=16),
    "c3s": ConfigSpec("c3s", "config 3 at 48^2 / 40^2 (generalised pencils), r=3, GMRES(40)",
                      r=3, seed=0, kmax=150, restart=40, flexible=False, npairs=10),
    "c3m": ConfigSpec("c3m", "config 3 at 250^2 / 175^2 with config 3's own shifts, r=3, GMRES(40)",
                      r=3, seed=0, kmax=8, restart=40, flexible=False, npairs=10,
                      extra={"shifts": "c3"}),
    "c5s": ConfigSpec("c5s", "config 5 family at 16^3 / 13^3, r=4, GMRES(30)",
                      r=4, seed=0, kmax=400, restart=30, flexible=False, npairs=16),
}

_BUILDERS = {"c1": _c1_matrices, "c2": _c2_matrices, "c3": _c3_matrices,
             "c5": _c5_matrices, "c3s": _c3s_matrices, "c5s": _c5s_matrices,
             "c3m": _c3m_matrices}


def build_problem(name, **sizes):
    """(A, B, M, C, f, g) for an ADI configuration (scipy CSR, numpy)."""
    spec = CONFIGS[name]
    A, B, M, C = _BUILDERS[name](**sizes)
    f, g = random_rhs(A.shape[0], B.shape[0], spec.r, spec.seed)
    return A, B, M, C, f, g


def build_c4(n0=4096, r=8, seed=0):
    """Config 4 operator and an n x r Gaussian block (Philox(seed))."""
    A = _c4_matrix(n0)
    gen = np.random.Generator(np.random.Philox(seed))
    X = gen.standard_normal((A.shape[0], r))
    return A, X
