"""Where does the end-to-end run() time go (config 2)?"""
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


def once():
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
    sol, rep = pb.run(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible)
    return sol.Z, sol.Y


for _ in range(2):
    once()
torch.cuda.synchronize()
t0 = time.perf_counter()
once()
print("e2e", time.perf_counter() - t0)
pr = cProfile.Profile()
pr.enable()
once()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
