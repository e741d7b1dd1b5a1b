"""Sweep engine knobs on config 2 (device-resident ADI), print one line each.

    python tools/tune_c2.py [--reps 3]
"""
import argparse
import itertools
import os
import sys
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2312_02891_b200 as pb  # noqa: E402
from paper_2312_02891_b200 import _lib, configs as cfgs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--config", default="c2")
    args = ap.parse_args()
    spec = cfgs.CONFIGS[args.config]
    A, B, M, C, f, g = cfgs.build_problem(args.config)
    pairs, cyclic = spec.load_shift_pairs()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
    cfg = pb.AdiConfig(strategy=spec.strategy, kmax=spec.kmax, precond_kind_A="jacobi",
                       precond_kind_B="jacobi")
    seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
    warnings.simplefilter("ignore")
    for engine, conc, mepth, direct in itertools.product(["persistent"], [True, False],
                                                         [2], [0, 1]):
        eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                           concurrent=conc, engine=engine)
        eng.warm()
        eng.run()
        for b in (eng.bA, eng.bB):
            for ws in b._workspaces.values():
                ws.set_option(_lib.SAD_OPT_RESIDENT_CSR, direct)
                ws.set_option(_lib.SAD_OPT_MIN_ELEMS_PER_THREAD, mepth)
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, rep, _ = eng.run()
            ts.append(time.perf_counter() - t0)
        wss = list(eng.bA._workspaces.values()) + list(eng.bB._workspaces.values())
        for ws in wss:
            ws.profile(True)
        eng.run()
        prof = sum(ws.profile(False) for ws in wss)
        print(f"engine={engine} concurrent={conc} min_elems={mepth} resident_csr={direct}: solve {min(ts)*1e3:.1f} ms "
              f"(steps {rep.outer_iterations}, inner {rep.sum_inner_A}/{rep.sum_inner_B}) "
              f"kernel {prof[0]:.1f} ms, {prof[2]/prof[0]/1e6:.0f} GB/s, phaseA {prof[3]:.1f} "
              f"phaseC {prof[5]:.1f} cycle-end {prof[6]:.1f} ms, steps {int(prof[4])} | "
              f"workA {prof[8]:.1f} workC {prof[9]:.1f} finA {prof[10]:.1f} finC {prof[11]:.1f}",
              flush=True)
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                       engine="multi")
    eng.warm()
    eng.run()
    t0 = time.perf_counter()
    eng.run()
    print(f"engine=multi: solve {(time.perf_counter()-t0)*1e3:.1f} ms")


if __name__ == "__main__":
    main()
