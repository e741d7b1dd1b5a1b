"""Generate a config's shift file on the GPU (device Ritz values + the greedy
picker) and compare with a pinned file when one exists.

    python tools/gen_shifts.py c5 [--out configs/shifts_c5.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2312_02891_b200 import configs as cfgs  # noqa: E402
from paper_2312_02891_b200 import shifts as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--out", default=None)
    ap.add_argument("--rtol", type=float, default=1e-12)
    args = ap.parse_args()
    spec = cfgs.CONFIGS[args.config]
    t0 = time.perf_counter()
    A, B, M, C, f, g = cfgs.build_problem(args.config)
    t_build = time.perf_counter() - t0
    stats = {}
    t0 = time.perf_counter()
    rA = S.pencil_ritz_sets(A, M, source="A-side", rtol=args.rtol, stats=stats)
    tA = time.perf_counter() - t0
    rB = S.pencil_ritz_sets(B, C, source="B-side", rtol=args.rtol, stats=stats)
    tB = time.perf_counter() - t0 - tA
    seq = S.heuristic_shifts(rA, rB, npairs=spec.npairs)
    out = {"config": args.config, "n": A.shape[0], "m": B.shape[0], "build_s": t_build,
           "ritz_A_s": tA, "ritz_B_s": tB, "solves": stats, "npairs": spec.npairs,
           "distinct_pairs": len(set(seq.pairs)),
           "complex_pairs": sum(1 for a, b in seq.pairs if a.imag or b.imag),
           "ritz_A": [[z.real, z.imag] for z in np.concatenate([rA[0].values, rA[1].values])],
           "ritz_B": [[z.real, z.imag] for z in np.concatenate([rB[0].values, rB[1].values])]}
    if os.path.exists(spec.shift_file):
        pinned, _ = spec.load_shift_pairs()
        out["max_rel_diff_vs_pinned"] = max(
            max(abs(a - pa) / abs(pa), abs(b - pb) / abs(pb))
            for (a, b), (pa, pb) in zip(seq.pairs, pinned))
    if args.out:
        seq.to_json(args.out)
        out["written"] = args.out
    print(json.dumps(out))


if __name__ == "__main__":
    main()
