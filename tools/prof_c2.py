"""One warm config-2 ADI solve (for ncu captures of k_gmres_persistent)."""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2312_02891_b200 as pb  # noqa: E402
from paper_2312_02891_b200 import configs as cfgs  # noqa: E402

warnings.simplefilter("ignore")
spec = cfgs.CONFIGS["c2"]
A, B, M, C, f, g = cfgs.build_problem("c2")
pairs, cyclic = spec.load_shift_pairs()
prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
cfg = pb.AdiConfig(strategy=spec.strategy, kmax=int(os.environ.get("KMAX", spec.kmax)),
                   precond_kind_A="jacobi", precond_kind_B="jacobi")
eng = pb.DeviceAdi(prob, cfg, pb.ShiftSequence(pairs=pairs, cyclic=cyclic),
                   restart=spec.restart, flexible=spec.flexible, concurrent=False)
eng.warm()
_, rep, _ = eng.run()
print("steps", rep.outer_iterations, "converged", rep.converged)
