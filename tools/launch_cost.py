"""Host cost of one persistent-solve launch+finish pair on a tiny system
(config-1 A side, r=1, loose tolerance): the per-outer-step overhead floor."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_02891_b200 import GpuGmresBinding, configs as cfgs  # noqa: E402

A, B, _, _, f, g = cfgs.build_problem("c1")
b = GpuGmresBinding("A", A, None, restart=30)
rhs = torch.from_numpy(f.astype(np.complex128)).cuda()
x = torch.empty_like(rhs)
res = torch.empty_like(rhs)
for _ in range(20):
    tok = b.begin_device(-500.0, rhs, 1e3, x, res)
    b.end_device(tok)
torch.cuda.synchronize()
t0 = time.perf_counter()
N = 500
for _ in range(N):
    tok = b.begin_device(-500.0, rhs, 1e3, x, res)
    b.end_device(tok)
print(f"launch+finish of a trivial persistent solve: {1e6*(time.perf_counter()-t0)/N:.1f} us")
