"""Host-side cost of the device-resident ADI loop on config 2 (cProfile of one
warm DeviceAdi.run(), sorted by own time)."""
import cProfile
import os
import pstats
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_02891_b200 as pb  # noqa: E402
from paper_2312_02891_b200 import configs as cfgs  # noqa: E402

warnings.simplefilter("ignore")
spec = cfgs.CONFIGS["c2"]
A, B, M, C, f, g = cfgs.build_problem("c2")
pairs, cyclic = spec.load_shift_pairs()
prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
cfg = pb.AdiConfig(strategy=spec.strategy, kmax=spec.kmax, precond_kind_A="jacobi",
                   precond_kind_B="jacobi")
seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible)
eng.warm()
for _ in range(3):
    eng.run()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
eng.run()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
