"""Time LowRankSolution._stack on factor shapes of configs 3 and 5 (synthetic device blocks).

    python tools/download_bench.py [c3|c5]
"""
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_02891_b200.adi import LowRankSolution  # noqa: E402

SHAPES = {"c3": (1_000_000, 3, 95), "c3y": (490_000, 3, 95), "c5": (8_000_000, 4, 77),
          "c5y": (4_096_000, 4, 77)}
for name in sys.argv[1:] or ["c3", "c3y"]:
    rows, r, k = SHAPES[name]
    z = torch.randn(k, rows, r, dtype=torch.complex128, device="cuda")
    blocks = [z[i] for i in range(k)]
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        out = LowRankSolution._stack(blocks, rows, r)
        dt = time.perf_counter() - t0
        gb = out.nbytes / 1e9
        print(f"{name} rep {rep}: {gb:.2f} GB in {dt:.2f} s = {gb / dt:.1f} GB/s", flush=True)
        chk = abs(out[rows // 2, 5 * r + 1] - complex(z[5, rows // 2, 1].cpu())) == 0
        assert chk
        del out
