"""Config 2, A/B concurrent: share of the SMs given to the A side."""
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
SPLITS = [None if x == "none" else float(x) for x in os.environ.get("SPLITS", "none,0.85").split(",")]
for split in SPLITS:
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                       sm_split=split)
    eng.warm()
    for _ in range(2):
        eng.run()
    ts = []
    for _ in range(int(os.environ.get("REPS", "5"))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, rep, _ = eng.run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"split={split}: min {ts[0]:.1f} median {ts[len(ts) // 2]:.1f} ms (inner {rep.sum_inner_A}/{rep.sum_inner_B})", flush=True)
    del eng
