"""Golden for the config-4 fixed-step parity test at 1024^2:
the oracle's per-column TRUE residual norms after 100 fixed Jacobi-GMRES(100)
steps on the config-4 operator family at n0 = 1024 (1,048,576 rows), r = 8
Gaussian columns (Philox(0), configs.build_c4), lambda_max from the reference's
own arnoldi_ritz (10 steps from ones) as configs/make_shift_c4.py.  Config 4's
own shift 0.1 * lambda_max makes the shifted operator so well conditioned
(kappa ~ 12) that 100 steps end at round-off (true residuals ~1e-13, nothing to
compare), so the parity golden uses shift = 0.001 * lambda_max (kappa ~ 1e3):
100 steps leave a residual of order 1e-3 ||b||, a well-determined number.
Both orthogonalisation variants of the oracle (CGS2 and the delayed-Gram DCGS2
of the device engine) are stored.

Run in the build container (the reference must be importable):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden_c4.py

Takes ~10 minutes of CPU (the oracle is a per-column numpy loop).
"""
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

N0, R, STEPS = 1024, 8, 100


def _shift():
    from sylvadi.shifts import arnoldi_ritz          # the reference
    from paper_2312_02891_b200.configs import _c4_matrix
    A = _c4_matrix(N0)
    ritz = arnoldi_ritz(lambda x: A @ x, np.ones(A.shape[0]), 10)
    lam = complex(ritz.values[np.argmax(np.abs(ritz.values))])
    return 0.001 * lam.real


def _column(args):
    orth, c, shift = args
    from oracle import sylvadi_oracle as orc
    from paper_2312_02891_b200.configs import build_c4
    A, X = build_c4(N0, R, 0)
    ob = orc.Binding("A", A, None, solver="gmres", restart=STEPS, max_iterations=STEPS,
                     orth=orth)
    out = ob.solve(shift, X[:, c:c + 1].copy(), 1e-300)
    return orth, c, float(out.achieved_residual_norms[0]), int(out.iterations[0])


def main():
    shift = _shift()
    jobs = [(o, c, shift) for o in ("cgs2", "dcgs2") for c in range(R)]
    res = {"cgs2": np.zeros(R), "dcgs2": np.zeros(R)}
    with ProcessPoolExecutor(max_workers=int(os.environ.get("WORKERS", "8"))) as ex:
        for orth, c, nrm, it in ex.map(_column, jobs):
            assert it == STEPS
            res[orth][c] = nrm
            print(orth, c, nrm, flush=True)
    np.savez(os.path.join(HERE, "oracle_c4_1024_fixed.npz"), n0=N0, r=R, steps=STEPS,
             shift=shift, cgs2=res["cgs2"], dcgs2=res["dcgs2"])
    print("shift", shift, "max rel diff cgs2/dcgs2",
          np.max(np.abs(res["cgs2"] - res["dcgs2"]) / res["cgs2"]))


if __name__ == "__main__":
    main()
