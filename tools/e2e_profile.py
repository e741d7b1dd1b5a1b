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

# phase breakdown (wall clock, synchronised)
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    sol, rep, st = eng.run()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    Z = sol.Z
    t3 = time.perf_counter()
    Y = sol.Y
    t4 = time.perf_counter()
    print(f"phases: construct {1e3*(t1-t0):.1f} ms, run {1e3*(t2-t1):.1f} ms, "
          f"Z {1e3*(t3-t2):.1f} ms ({Z.nbytes/1e6:.0f} MB), Y {1e3*(t4-t3):.1f} ms")

# first run of a fresh engine vs a second run of the same (warm) engine
for _ in range(3):
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible)
    ts = []
    for _k in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sol, rep, st = eng.run()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    print("fresh engine runs (ms):", [round(x, 1) for x in ts])
pr = cProfile.Profile()
prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible)
pr.enable()
eng.run()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
