"""Per-step phase times of the persistent kernel on config 2 (block 0's work
before each grid barrier, the reducing block's serial finisher sections, the
phase-A SpMM), in microseconds per Arnoldi step."""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_02891_b200 as pb  # noqa: E402
from paper_2312_02891_b200 import _lib, configs as cfgs  # noqa: E402

warnings.simplefilter("ignore")
name = os.environ.get("CFG", "c2")
spec = cfgs.CONFIGS[name]
A, B, M, C, f, g = cfgs.build_problem(name)
pairs, cyclic = spec.load_shift_pairs()
prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
cfg = pb.AdiConfig(strategy=spec.strategy, kmax=int(os.environ.get("KMAX", spec.kmax)),
                   precond_kind_A="jacobi",
                   precond_kind_B="jacobi")
seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
CONC = [c == "1" for c in os.environ.get("CONC", "1,0").split(",")]
PHASE = os.environ.get("PHASE", "direct,tma").split(",")
for conc in CONC:
    for phase_a in PHASE:
        eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                           concurrent=conc, phase_a=phase_a)
        eng.warm()
        eng.run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.run()
        e1.record()
        torch.cuda.synchronize()
        for side, b in (("A", eng.bA), ("B", eng.bB)):
            wss = list(b._workspaces.values())
            for ws in wss:
                ws.profile(True)
        eng.run()
        for side, b in (("A", eng.bA), ("B", eng.bB)):
            p = sum(ws.profile(False) for ws in b._workspaces.values())
            st = max(p[4], 1)
            us = 1e3 / st
            print(f"concurrent={conc} phase_a={phase_a} side {side}: solve {e0.elapsed_time(e1):.1f} ms | "
                  f"steps {int(p[4])} kernel {p[0]:.1f} ms | per step: phaseA {p[3]*us:.1f} "
                  f"phaseC {p[5]*us:.1f} us | workA {p[8]*us:.1f} spmmA {p[12]*us:.1f} finA {p[10]*us:.1f} "
                  f"workC {p[9]*us:.1f} finC {p[11]*us:.1f} us", flush=True)
