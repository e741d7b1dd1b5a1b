"""One device-resident ADI solve of a BASELINE configuration, with the GPU
true-residual check.  Prints one JSON line.

    python tools/run_config.py c3 [--kmax K] [--no-verify]
"""
import argparse
import json
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_02891_b200 as pb  # noqa: E402
from paper_2312_02891_b200 import configs as cfgs  # noqa: E402
from paper_2312_02891_b200.verify import true_residual_norm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--kmax", type=int, default=None)
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--sequential", action="store_true", help="A and B solves one after the other")
    ap.add_argument("--concurrent", action="store_true", help="A and B solves overlapped")
    ap.add_argument("--phase-a", default="auto", choices=["auto", "tma", "direct"])
    ap.add_argument("--profile", action="store_true", help="instrumented pass (GB/s per kernel)")
    ap.add_argument("--engine", default="persistent", choices=["persistent", "multi", "rowpart"])
    args = ap.parse_args()
    warnings.simplefilter("ignore")
    spec = cfgs.CONFIGS[args.config]
    t0 = time.perf_counter()
    A, B, M, C, f, g = cfgs.build_problem(args.config)
    t_build = time.perf_counter() - t0
    pairs, cyclic = spec.load_shift_pairs()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
    cfg = pb.AdiConfig(strategy=spec.strategy, kmax=args.kmax or spec.kmax,
                       precond_kind_A="jacobi", precond_kind_B="jacobi")
    seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
    t0 = time.perf_counter()
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                       concurrent=False if args.sequential else (True if args.concurrent else "auto"),
                       phase_a=args.phase_a, engine=args.engine)
    eng.warm()
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    walls = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sol, rep, _ = eng.run()
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    out = {"config": args.config, "n": prob.n, "m": prob.m, "r": prob.r,
           "nnz_A": int(A.nnz), "nnz_B": int(B.nnz), "restart": spec.restart,
           "flexible": spec.flexible, "kmax": cfg.kmax, "outer_steps": rep.outer_iterations,
           "converged": rep.converged, "final_scaled_residual": rep.final_scaled_residual,
           "sum_inner_A": rep.sum_inner_A, "sum_inner_B": rep.sum_inner_B,
           "wall_s": min(walls), "walls_s": walls, "build_s": t_build, "setup_s": t_setup,
           "dtype": str(sol.device_blocks[0][0].dtype) if sol.steps else None,
           "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}
    if args.profile:
        wss = list(eng.bA._workspaces.values()) + list(eng.bB._workspaces.values())
        for ws in wss:
            ws.profile(True)
        eng.run()
        tot = np.zeros(13)
        for ws in wss:
            tot += ws.profile(False)
        out["profile"] = {"kernel_ms": tot[0], "launches": int(tot[1]),
                          "algorithmic_GBps": tot[2] / (tot[0] * 1e-3) / 1e9,
                          "phaseA_ms": tot[3], "arnoldi_steps": int(tot[4]),
                          "phaseC_ms": tot[5], "cycle_end_ms": tot[6], "cycles": int(tot[7]),
                          "workA_ms": tot[8], "workC_ms": tot[9], "finA_ms": tot[10],
                          "finC_ms": tot[11], "spmmA_ms": tot[12]}
    if not args.no_verify:
        t0 = time.perf_counter()
        trn = true_residual_norm(prob, sol)
        out["true_residual_norm"] = trn
        out["true_scaled_residual"] = trn / rep.rhs_norm
        out["verify_s"] = time.perf_counter() - t0
    print(json.dumps(out))
    steps = [(r.step, r.inner_it_A, r.inner_it_B, r.scaled_res) for r in rep.records]
    print(json.dumps({"per_step": steps}))


if __name__ == "__main__":
    main()
