"""Stand-alone SpMM timing with and without the banded plan on a configuration's operators.

    python tools/spmm_band_probe.py c3 [r]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_02891_b200 import configs as cfgs  # noqa: E402
from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator  # noqa: E402

name = sys.argv[1]
A, B, M, C, f, g = cfgs.build_problem(name)
r = int(sys.argv[2]) if len(sys.argv) > 2 else f.shape[1]
pairs, _ = cfgs.CONFIGS[name].load_shift_pairs()
shift = complex(pairs[0][1])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cplx in (True, False):
    if not cplx and shift.imag != 0:
        sh = shift.real
    else:
        sh = shift
    for band in ("1", "0"):
        os.environ["SAD_SPMM_BAND"] = band
        dm = DeviceMatrix(A)
        dmm = None if M is None else DeviceMatrix(M)
        op = DeviceOperator(dm, dmm, sh if cplx else complex(sh).real, precond_kind="jacobi")
        n = A.shape[0]
        x = torch.randn(n, r, dtype=torch.complex128 if cplx else torch.float64, device="cuda")
        y = torch.empty_like(x)
        info = op.band_info()
        for _ in range(3):
            op.apply(x, y)
        ts = []
        for _ in range(5):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); op.apply(x, y); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        esz = 16 if cplx else 8
        vsz = 16 if (cplx and complex(sh).imag != 0 and M is not None) else 8
        nnz = A.nnz if M is None else (A + M).nnz
        alg = nnz * (vsz + 4) + 4 * (n + 1) + 2 * esz * r * n
        print(f"{name} r={r} complex={cplx} band={band} plan={info}: {np.mean(ts)*1e3:.1f} us, "
              f"{alg / np.mean(ts) / 1e6:.0f} GB/s algorithmic", flush=True)
        del op, dm, dmm
