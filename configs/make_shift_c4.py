"""Pin config 4's shift: alpha = 0.1 * lambda, lambda the
largest-magnitude Ritz value of 10 Arnoldi steps of the config-4 operator
(the reference's own arnoldi_ritz, shifts.py:70-98, start vector ones as
pencil_ritz_sets, shifts.py:111).  Run in the build container, where
/root/reference is importable:

    PYTHONPATH=/root/reference/pkg/src:. python configs/make_shift_c4.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def main(n0=4096, steps=10):
    from sylvadi.shifts import arnoldi_ritz          # the reference
    from paper_2312_02891_b200.configs import _c4_matrix
    A = _c4_matrix(n0)
    ritz = arnoldi_ritz(lambda x: A @ x, np.ones(A.shape[0]), steps)
    lam = complex(ritz.values[np.argmax(np.abs(ritz.values))])
    out = {"n0": n0, "arnoldi_steps": steps, "lambda_max": [lam.real, lam.imag],
           "shift": 0.1 * lam.real,
           "how": "sylvadi.shifts.arnoldi_ritz(A @ x, ones, 10); shift = 0.1 * Re(lambda_max)"}
    with open(os.path.join(HERE, "shift_c4.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(out)


if __name__ == "__main__":
    main()
