"""Config 2: per-step wall times (CUDA events) of repeated device-resident
solves, with and without an L2 flush before each, A/B concurrent and not."""
import os
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
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for conc in (True, False):
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                       concurrent=conc)
    eng.warm()
    for _ in range(3):
        eng.run()
    for do_flush in (False, True):
        ts = []
        for _ in range(8):
            if do_flush:
                flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            eng.run()
            e1.record()
            torch.cuda.synchronize()
            ts.append(round(e0.elapsed_time(e1), 1))
        print(f"concurrent={conc} flush={do_flush}: {ts}", flush=True)
