"""Config 2: persistent-kernel grid sizing (min elements per thread) sweep."""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_02891_b200 as pb  # noqa: E402
from paper_2312_02891_b200 import _lib, configs as cfgs  # noqa: E402

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
eng.run()
for mept in (1, 2, 3, 4, 5, 6, 8):
    for b in (eng.bA, eng.bB):
        for ws in b._workspaces.values():
            ws.set_option(_lib.SAD_OPT_MIN_ELEMS_PER_THREAD, mept)
    eng.run()
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, rep, _ = eng.run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"min_elems_per_thread={mept}: {min(ts):.1f} ms (inner {rep.sum_inner_A}/{rep.sum_inner_B})",
          flush=True)
