"""Where does DeviceAdi construction + first-run operator creation go (config 2)?"""
import cProfile
import os
import pstats
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
for _ in range(2):
    pb.run(pb.SylvesterProblem(A=A, B=B, f=f, g=g), cfg, seq, restart=spec.restart,
           flexible=spec.flexible)
torch.cuda.synchronize()


def build():
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible)
    eng.warm()
    torch.cuda.synchronize()
    return eng


t0 = time.perf_counter()
build()
print("construct+warm", 1e3 * (time.perf_counter() - t0), "ms")
pr = cProfile.Profile()
pr.enable()
build()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
