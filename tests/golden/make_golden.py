"""Generate the golden fixtures by running the REFERENCE (build container only).

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [--with-c2]

Imports ``sylvadi`` from /root/reference/pkg/src (read-only) and writes:

* configs/shifts_c1.json, configs/shifts_c2.json -- the reference's own
  heuristic shifts (shifts.py:107-217) for configs 1 and 2, pinned so the
  oracle, the GPU runs and the CPU baselines share bit-identical shifts
  (the reference CLI does the same, cli.py:163-176);
* tests/golden/problem_hashes.json -- sha256 of the reference's
  convdiff_matrix / random_rhs outputs for the FD configs (pins
  paper_2312_02891_b200.problems);
* tests/golden/ref_small.npz -- reference outputs on small seeded cases:
  ShiftedOperator.apply (plain/adjoint, identity/sparse mass, real/complex
  shift), Jacobi dinv, bicgstab, tolerance strategies, residual norms;
* tests/golden/ref_c1_<strategy>_bicgstab.csv -- per-step records of the
  reference's run_with_state on config 1 with Jacobi-BiCGstab (its own inner
  path), kmax=150;
* tests/golden/refdriver_c1_gmres.csv -- the reference's run_with_state driving
  the oracle's GMRES(50) binding on config 1 (pins the oracle's driver
  restatement when paired with GMRES);
* tests/golden/oracle_c1_gmres.csv (and _c2 with --with-c2) -- the oracle's
  own GMRES ADI run, the per-step iteration counts the GPU must match (+-2).

/root/reference is never read at test, smoke or bench time.
"""

import argparse
import hashlib
import json
import os
import sys
import warnings

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import sylvadi as sv  # noqa: E402  (the reference)

from oracle import sylvadi_oracle as orc  # noqa: E402
from paper_2312_02891_b200 import configs as cfgs  # noqa: E402

GOLD = os.path.join(REPO, "tests", "golden")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def ref_c1():
    A = sv.convdiff_matrix(sv.ConvDiffSpec(2, 64, (lambda x, y: 10.0 * x,
                                                   lambda x, y: 10.0 * y)))
    B = sv.convdiff_matrix(sv.ConvDiffSpec(2, 48, (lambda x, y: 50.0 * y,
                                                   lambda x, y: -50.0 * x)))
    f, g = sv.random_rhs(A.nrows, B.nrows, 1, 0)
    return A, B, f, g


def ref_c2():
    A = sv.convdiff_matrix(sv.ConvDiffSpec(3, 40, (20.0, 20.0, 20.0)))
    B = sv.convdiff_matrix(sv.ConvDiffSpec(3, 30, (lambda x, y, z: 5.0 * x,
                                                   lambda x, y, z: -5.0 * y,
                                                   lambda x, y, z: 5.0 * z)))
    f, g = sv.random_rhs(A.nrows, B.nrows, 2, 0)
    return A, B, f, g


def make_shifts(name, A, B, npairs):
    path = os.path.join(REPO, "configs", f"shifts_{name}.json")
    if os.path.exists(path):
        print("keep", path)
        return sv.ShiftSequence.from_json(path)
    seq = sv.heuristic_shifts(sv.pencil_ritz_sets(A), sv.pencil_ritz_sets(B),
                              npairs=npairs)
    os.makedirs(os.path.dirname(path), exist_ok=True)
    seq.to_json(path)
    print("wrote", path)
    return seq


def problem_hashes():
    out = {}
    for name, builder in (("c1", ref_c1), ("c2", ref_c2)):
        A, B, f, g = builder()
        out[name] = {
            "A": sha(A.offsets.astype(np.int64), A.indices.astype(np.int64), A.values),
            "B": sha(B.offsets.astype(np.int64), B.indices.astype(np.int64), B.values),
            "f": sha(f), "g": sha(g),
            "nnzA": int(A.nnz), "nnzB": int(B.nnz),
        }
    # a tiny case with zero convection and one with constant convection
    for tag, spec in (("lap3_5", sv.ConvDiffSpec(3, 5, None)),
                      ("cd2_7", sv.ConvDiffSpec(2, 7, (3.0, -2.0)))):
        M = sv.convdiff_matrix(spec)
        out[tag] = {"A": sha(M.offsets.astype(np.int64), M.indices.astype(np.int64),
                             M.values)}
    with open(os.path.join(GOLD, "problem_hashes.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote problem_hashes.json")


def small_cases():
    rng = np.random.default_rng(20260826)
    data = {}

    def rand_sparse(n, density=0.3):
        d = rng.standard_normal((n, n))
        d[rng.random((n, n)) > density] = 0.0
        d += np.diag(4.0 + rng.random(n))
        return d

    n = 9
    base = rand_sparse(n)
    mass = rand_sparse(n)
    x = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
    data["base"], data["mass"], data["x"] = base, mass, x
    for tag, shift in (("real", -1.7 + 0j), ("cplx", -2.0 + 0.4j)):
        for adj in (False, True):
            for mname, m in (("I", None), ("M", mass)):
                op = sv.ShiftedOperator(sv.SparseMatrix(base),
                                        None if m is None else sv.SparseMatrix(m),
                                        shift, adjoint=adj)
                key = f"apply_{tag}_{'adj' if adj else 'fwd'}_{mname}"
                data[key] = op.apply(x)
                fact = sv.factorize(op.assembled(), "jacobi")
                data["dinv_" + key[6:]] = fact._diag_inv
    # bicgstab on a diagonally dominant unsymmetric system, jacobi
    nb = 40
    dense = rng.standard_normal((nb, nb))
    dense += np.diag(np.abs(dense).sum(axis=1) + 1.0)
    b = rng.standard_normal((nb, 2))
    op = sv.ShiftedOperator(sv.SparseMatrix(dense), None, -0.5 + 0.25j)
    fact = sv.factorize(op.assembled(), "jacobi")
    res = sv.bicgstab(sv.InnerSolveRequest(op, b, 1e-10, preconditioner=fact))
    data["bicg_dense"], data["bicg_b"] = dense, b
    data["bicg_x"], data["bicg_iters"] = res.solution, res.iterations
    data["bicg_norms"] = res.achieved_residual_norms
    # tolerance strategies over a grid
    rows = []
    for strat in ("fixed", "dynamic_mid", "dynamic_mid_bl", "dynamic_b",
                  "dynamic_b_bl", "direct_a_iter_b", "iter_a_direct_b"):
        cfg = sv.AdiConfig(strategy=strat, gap_budget=3e-7, kmax=40)
        for k in (1, 2, 7):
            for (uu, vv) in ((0.0, 0.0), (1e-10, 3e-11)):
                eh = sv.tolerance_budget(cfg, k, uu, vv)
                for nw, nt in ((1.0, 2.0), (3e-4, 1e-6), (5e-9, 2e-3)):
                    dec = sv.choose_tolerances(cfg, k, nw, nt, eh)
                    rows.append([eh, dec.delta_A, dec.delta_B,
                                 float(dec.clamped_A_min), float(dec.clamped_B_min)])
    data["tol_table"] = np.array(rows)
    # residual norms
    w = rng.standard_normal((30, 3)) + 1j * rng.standard_normal((30, 3))
    t = rng.standard_normal((20, 3)) + 1j * rng.standard_normal((20, 3))
    data["crn_w"], data["crn_t"] = w, t
    data["crn"] = np.array([sv.computed_residual_norm(w, t)])
    np.savez_compressed(os.path.join(GOLD, "ref_small.npz"), **data)
    print("wrote ref_small.npz")


def write_csv(path, report):
    rows = ["step,scaled_res,delta_A,delta_B,achieved_rA,achieved_rB,"
            "inner_it_A,inner_it_B,u,v"]
    for rec in report.records:
        rows.append(f"{rec.step},{rec.scaled_res:.16e},{rec.delta_A:.16e},"
                    f"{rec.delta_B:.16e},{rec.achieved_rA:.16e},"
                    f"{rec.achieved_rB:.16e},{rec.inner_it_A},{rec.inner_it_B},"
                    f"{rec.u:.16e},{rec.v:.16e}")
    with open(path, "w") as fh:
        fh.write("\n".join(rows) + "\n")
    print("wrote", path)


class OracleGmresBinding:
    """Adapter: the oracle's GMRES behind the reference's SolverBinding seam."""

    def __init__(self, side, base, restart, flexible=False):
        self.inner = orc.Binding(side, base.scipy(), None,
                                 solver="fgmres" if flexible else "gmres",
                                 restart=restart)

    def solve(self, shift, rhs, delta):
        return self.inner.solve(shift, rhs, delta)


def c1_runs(seq):
    A, B, f, g = ref_c1()
    problem = sv.SylvesterProblem(A=A, B=B, f=f, g=g)
    for strat in ("dynamic_mid_bl", "fixed"):
        cfg = sv.AdiConfig(strategy=strat, kmax=150, precond_kind_A="jacobi",
                           precond_kind_B="jacobi")
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            _, rep, _ = sv.run_with_state(problem, cfg, seq)
        write_csv(os.path.join(GOLD, f"ref_c1_{strat}_bicgstab.csv"), rep)
    # reference driver + oracle GMRES
    cfg = sv.AdiConfig(strategy="dynamic_mid_bl", kmax=150)
    bind = sv.adi.SolverBindings(A=OracleGmresBinding("A", A, 50),
                                 B=OracleGmresBinding("B", B, 50))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, rep, _ = sv.run_with_state(problem, cfg, seq, bindings=bind)
    write_csv(os.path.join(GOLD, "refdriver_c1_gmres.csv"), rep)


def oracle_run(name):
    spec = cfgs.CONFIGS[name]
    A, B, M, C, f, g = cfgs.build_problem(name)
    pairs, cyclic = spec.load_shift_pairs()
    ocfg = orc.Config(strategy=spec.strategy, kmax=spec.kmax,
                      outer_tolerance=spec.outer_tolerance)
    solver = "fgmres" if spec.flexible else "gmres"
    bA = orc.Binding("A", A, M, solver=solver, restart=spec.restart)
    bB = orc.Binding("B", B, C, solver=solver, restart=spec.restart)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        run = orc.run_adi(A, B, f, g, ocfg, pairs, bA, bB, M=M, C=C, cyclic=cyclic)
    with open(os.path.join(GOLD, f"oracle_{name}_gmres.csv"), "w") as fh:
        fh.write(orc.steps_csv(run))
    print(f"oracle {name}: {run.outer_iterations} steps, converged={run.converged},"
          f" sum inner {run.sum_inner_A}/{run.sum_inner_B}, {run.wall_ms/1e3:.1f}s")


def make_shifts_generalised(name, A, M, B, C, npairs):
    """Reference heuristic shifts for pencils (A, M), (B, C) (shifts.py:107-132)."""
    path = os.path.join(REPO, "configs", f"shifts_{name}.json")
    if os.path.exists(path):
        print("keep", path)
        return
    to = lambda X: None if X is None else sv.SparseMatrix(X)
    seq = sv.heuristic_shifts(sv.pencil_ritz_sets(to(A), to(M)),
                              sv.pencil_ritz_sets(to(B), to(C)), npairs=npairs)
    seq.to_json(path)
    print("wrote", path)


def small_configs():
    """Reduced configs 3 and 5: reference shifts + oracle GMRES goldens."""
    for name in ("c3s", "c5s"):
        A, B, M, C, f, g = cfgs.build_problem(name)
        make_shifts_generalised(name, A, M, B, C, cfgs.CONFIGS[name].npairs)
        oracle_run(name)
    # the reference's own driver on the generalised small config (BiCGstab):
    # pins the mass-matrix handling of the oracle driver (adi.py:520-528)
    A, B, M, C, f, g = cfgs.build_problem("c3s")
    seq = sv.ShiftSequence.from_json(os.path.join(REPO, "configs", "shifts_c3s.json"))
    problem = sv.SylvesterProblem(A=sv.SparseMatrix(A), B=sv.SparseMatrix(B), f=f, g=g,
                                  M=sv.SparseMatrix(M), C=sv.SparseMatrix(C))
    cfg = sv.AdiConfig(strategy="dynamic_mid_bl", kmax=150, precond_kind_A="jacobi",
                       precond_kind_B="jacobi")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        _, rep, _ = sv.run_with_state(problem, cfg, seq)
    write_csv(os.path.join(GOLD, "ref_c3s_dynamic_mid_bl_bicgstab.csv"), rep)


def verify_goldens():
    """The reference's true_residual_norm / residual_gap (adi.py:655-726) on
    short runs of its own driver: a standard pair (config 1, 6 steps) and a
    generalised pair (config 3 at 48^2 / 40^2, 4 steps).  Factors, gammas and
    the reference values go to tests/golden/ref_verify_<case>.npz."""
    cases = (("c1", 6), ("c3s", 4))
    for name, kmax in cases:
        A, B, M, C, f, g = cfgs.build_problem(name)
        seq = sv.ShiftSequence.from_json(os.path.join(REPO, "configs", f"shifts_{name}.json"))
        to = lambda X: None if X is None else sv.SparseMatrix(X)
        problem = sv.SylvesterProblem(A=to(A), B=to(B), f=f, g=g, M=to(M), C=to(C))
        cfg = sv.AdiConfig(strategy="dynamic_mid_bl", kmax=kmax, precond_kind_A="jacobi",
                           precond_kind_B="jacobi", keep_inner_residuals=True)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            sol, rep, state = sv.run_with_state(problem, cfg, seq)
        trn = sv.true_residual_norm(problem, sol)
        gap = sv.residual_gap(problem, state)
        fid = sv.verify_factor_identity(problem, state)
        path = os.path.join(GOLD, f"ref_verify_{name}.npz")
        np.savez_compressed(path, Z=sol.Z, Y=sol.Y, gdiag=sol.gamma_diag(),
                            true_residual_norm=trn, residual_gap=gap,
                            steps=rep.outer_iterations,
                            S_A=state.S_A(), S_B=state.S_B(), w=state.w, t=state.t,
                            gammas=np.asarray(state.gammas, dtype=complex),
                            shift_history=np.asarray(state.shift_history, dtype=complex),
                            u=state.u, v=state.v, factor_identity=fid)
        print(f"{path}: {rep.outer_iterations} steps, true residual {trn:.6e}, gap {gap:.6e}")


def ritz_goldens():
    """The reference's pencil_ritz_sets (shifts.py:101-129, splu-based) for the
    configs whose shifts are pinned; values go to tests/golden/ref_ritz.npz so
    the device Ritz generator and the host greedy picker can be checked
    against them (and against configs/shifts_<name>.json)."""
    out = {}
    to = lambda X: None if X is None else sv.SparseMatrix(X)
    for name in ("c1", "c2", "c3s", "c5s"):
        A, B, M, C, f, g = cfgs.build_problem(name)
        for side, (base, mass) in (("A", (A, M)), ("B", (B, C))):
            d, inv = sv.pencil_ritz_sets(to(base), to(mass))
            out[f"{name}_{side}_direct"] = d.values
            out[f"{name}_{side}_inverse"] = inv.values
        seq = sv.ShiftSequence.from_json(os.path.join(REPO, "configs", f"shifts_{name}.json"))
        al = [a for a, _ in seq.pairs]
        be = [b for _, b in seq.pairs]
        ra = np.concatenate([out[f"{name}_A_direct"], out[f"{name}_A_inverse"]])
        rb = np.concatenate([out[f"{name}_B_direct"], out[f"{name}_B_inverse"]])
        out[f"{name}_objective"] = sv.shift_objective(al, be, ra, rb)
        print(name, "ritz sets done")
    np.savez_compressed(os.path.join(GOLD, "ref_ritz.npz"), **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--with-c2", action="store_true")
    ap.add_argument("--small", action="store_true", help="only the reduced configs 3/5")
    ap.add_argument("--c3-shifts", action="store_true", help="full-size config-3 shifts")
    ap.add_argument("--verify", action="store_true", help="true_residual_norm goldens")
    ap.add_argument("--ritz", action="store_true", help="reference Ritz-set goldens")
    args = ap.parse_args()
    if args.ritz:
        ritz_goldens()
        return
    if args.verify:
        verify_goldens()
        return
    if args.small:
        small_configs()
        return
    if args.c3_shifts:
        A, B, M, C, f, g = cfgs.build_problem("c3")
        make_shifts_generalised("c3", A, M, B, C, cfgs.CONFIGS["c3"].npairs)
        return
    os.makedirs(GOLD, exist_ok=True)
    problem_hashes()
    small_cases()
    A, B, f, g = ref_c1()
    seq1 = make_shifts("c1", A, B, cfgs.CONFIGS["c1"].npairs)
    c1_runs(seq1)
    oracle_run("c1")
    if args.with_c2:
        A, B, f, g = ref_c2()
        make_shifts("c2", A, B, cfgs.CONFIGS["c2"].npairs)
        oracle_run("c2")


if __name__ == "__main__":
    main()
