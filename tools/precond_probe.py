"""Config 1 through the device driver with each preconditioner kind (BiCGstab
inner solver, droptol 0.1): wall time of one device-resident ADI run and the
inner iteration counts (profiles/r02/precond_c1_device_vs_cpu.txt)."""
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_02891_b200 as pb  # noqa: E402
from paper_2312_02891_b200 import configs as cfgs  # noqa: E402

warnings.simplefilter("ignore")
A, B, M, C, f, g = cfgs.build_problem("c1")
pairs, cyclic = cfgs.CONFIGS["c1"].load_shift_pairs()
for kind in ("jacobi", "ilut", "ilu0"):
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
    cfg = pb.AdiConfig(strategy="dynamic_mid_bl", kmax=150, precond_kind_A=kind,
                       precond_kind_B=kind, precond_droptol_A=0.1, precond_droptol_B=0.1)
    eng = pb.DeviceAdi(prob, cfg, pb.ShiftSequence(pairs=pairs, cyclic=cyclic), solver="reference")
    eng.warm()
    eng.run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol, rep, _ = eng.run()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"PC {kind}: device {dt:.3f} s ({rep.outer_iterations} steps, "
          f"inner {rep.sum_inner_A}/{rep.sum_inner_B})", flush=True)
