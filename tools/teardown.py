"""Config 2: host cost of SylvesterProblem construction and of the device
engine's teardown (operator / matrix destruction) around pb.run."""
import gc
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_02891_b200 as pb  # noqa: E402
from paper_2312_02891_b200 import configs as cfgs  # noqa: E402

warnings.simplefilter("ignore")
spec = cfgs.CONFIGS["c2"]
A, B, M, C, f, g = cfgs.build_problem("c2")
pairs, cyclic = spec.load_shift_pairs()
cfg = pb.AdiConfig(strategy=spec.strategy, kmax=spec.kmax, precond_kind_A="jacobi",
                   precond_kind_B="jacobi")
seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
for _ in range(3):
    t0 = time.perf_counter()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
    t1 = time.perf_counter()
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible)
    sol, rep, st = eng.run()
    Z, Y = sol.Z, sol.Y
    t2 = time.perf_counter()
    del eng, sol, st
    gc.collect()
    t3 = time.perf_counter()
    print(f"problem {1e3*(t1-t0):.1f} ms, construct+run+download {1e3*(t2-t1):.1f} ms, "
          f"teardown {1e3*(t3-t2):.1f} ms", flush=True)
