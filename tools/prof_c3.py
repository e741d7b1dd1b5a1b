"""A short device-resident config-3 ADI (KMAX outer steps, default 2) for ncu
captures of k_gmres_persistent on the HBM-bound generalised pencils."""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2312_02891_b200 as pb  # noqa: E402
from paper_2312_02891_b200 import configs as cfgs  # noqa: E402

warnings.simplefilter("ignore")
name = os.environ.get("CFG", "c3")
spec = cfgs.CONFIGS[name]
A, B, M, C, f, g = cfgs.build_problem(name)
pairs, cyclic = spec.load_shift_pairs()
prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
cfg = pb.AdiConfig(strategy=spec.strategy, kmax=int(os.environ.get("KMAX", 2)),
                   precond_kind_A="jacobi", precond_kind_B="jacobi")
solver = os.environ.get("SOLVER", "gmres")
eng = pb.DeviceAdi(prob, cfg, pb.ShiftSequence(pairs=pairs, cyclic=cyclic),
                   restart=spec.restart, flexible=spec.flexible, concurrent=False, solver=solver)
eng.warm()
_, rep, _ = eng.run()
print("steps", rep.outer_iterations, "inner", rep.sum_inner_A, rep.sum_inner_B)
