"""ADI-level parity on the GPU: the device-resident driver against the CPU
oracle on identical seeded inputs and pinned shifts (BASELINE north_star bars:
same outer step count, per-step inner iteration counts within +-2, final
relative residual below the outer tolerance, ||Z G Y^* - X_ref||_F/||X_ref||_F
<= 1e-8)."""

import os
import sys
import warnings

import numpy as np
import pytest

from oracle import sylvadi_oracle as orc
from paper_2312_02891_b200 import configs as cfgs

from conftest import GOLD, read_steps_csv

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _gpu_run(name, bindings_mode=False, **kw):
    import paper_2312_02891_b200 as pb
    spec = cfgs.CONFIGS[name]
    A, B, M, C, f, g = cfgs.build_problem(name)
    pairs, cyclic = spec.load_shift_pairs()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
    cfg = pb.AdiConfig(strategy=spec.strategy, kmax=spec.kmax,
                       outer_tolerance=spec.outer_tolerance,
                       precond_kind_A="jacobi", precond_kind_B="jacobi")
    seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
    bindings = None
    if bindings_mode:
        bindings = pb.make_gpu_bindings(prob, cfg, restart=spec.restart, flexible=spec.flexible)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return pb.run_with_state(prob, cfg, seq, bindings=bindings, restart=spec.restart,
                                 flexible=spec.flexible, **kw)


def _check_against_golden(rep, name):
    gold = read_steps_csv(os.path.join(GOLD, f"oracle_{name}_gmres.csv"))
    assert rep.converged
    assert rep.outer_iterations == len(gold)
    assert rep.final_scaled_residual < 1e-8
    worst = 0
    for rec, gd in zip(rep.records, gold):
        worst = max(worst, abs(rec.inner_it_A - gd["inner_it_A"]),
                    abs(rec.inner_it_B - gd["inner_it_B"]))
        assert abs(rec.delta_A - gd["delta_A"]) <= 1e-6 * gd["delta_A"] + 1e-300
    assert worst <= 2, worst
    return worst


def _oracle_run(name):
    """The oracle's own ADI run (same algorithm as the device: Jacobi GMRES /
    FGMRES with the delayed-Gram orthogonalisation) on the same seeded inputs."""
    spec = cfgs.CONFIGS[name]
    A, B, M, C, f, g = cfgs.build_problem(name)
    pairs, cyclic = spec.load_shift_pairs()
    ocfg = orc.Config(strategy=spec.strategy, kmax=spec.kmax)
    solver = "fgmres" if spec.flexible else "gmres"
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return orc.run_adi(A, B, f, g, ocfg, pairs,
                           orc.Binding("A", A, M, solver=solver, restart=spec.restart, orth="dcgs2"),
                           orc.Binding("B", B, C, solver=solver, restart=spec.restart, orth="dcgs2"),
                           M=M, C=C, cyclic=cyclic)


#: north_star: ||Z G Y^* - X_ref||_F / ||X_ref||_F <= 1e-8 in fp64
X_BAR = 1e-8


def _x_parity(name, sol):
    """X parity in factored form.  Default: against the committed sketch
    Omega^H X_ref of the oracle's own run (tests/golden/make_golden_x.py; an
    unbiased estimate of the Frobenius ratio).  SAD_FULL_ORACLE=1 runs the oracle
    here (minutes of CPU) and checks the exact quantity as well."""
    sys.path.insert(0, GOLD)
    import make_golden_x as mgx
    gold = np.load(os.path.join(GOLD, f"oracle_x_{name}.npz"))
    assert int(gold["steps"]) == len(sol.gammas)
    om = mgx.probes(sol.Z.shape[0], int(gold["k"]))
    got = mgx.sketch(sol.Z, sol.gammas, sol.r, sol.Y, om)
    err = float(np.linalg.norm(got - gold["sketch"]) / np.linalg.norm(gold["sketch"]))
    assert err <= X_BAR, err
    if os.environ.get("SAD_FULL_ORACLE") == "1":
        ref = _oracle_run(name)
        gd = np.repeat(np.asarray(sol.gammas), sol.r)
        gr = np.repeat(np.asarray(ref.gammas), sol.r)
        exact = orc.factored_relative_difference(sol.Z, gd, sol.Y, ref.Z, gr, ref.Y)
        assert exact <= X_BAR, exact
        print(f"X parity {name}: sketch {err:.3e} exact {exact:.3e}")
    return err


def test_c1_device_driver_matches_oracle():
    sol, rep, state = _gpu_run("c1")
    _check_against_golden(rep, "c1")
    _x_parity("c1", sol)


def test_c1_dropin_bindings_host_loop():
    """GpuGmresBinding behind the reference-style host loop (bindings=...)."""
    sol, rep, state = _gpu_run("c1", bindings_mode=True)
    _check_against_golden(rep, "c1")


def test_c1_multi_kernel_engine_matches_oracle():
    sol, rep, state = _gpu_run("c1", engine="multi")
    _check_against_golden(rep, "c1")


@pytest.mark.parametrize("engine", ["persistent", "multi"])
def test_c1_serial_and_concurrent_sides_agree(engine):
    _, rep1, _ = _gpu_run("c1", concurrent=False, engine=engine)
    _, rep2, _ = _gpu_run("c1", concurrent=True, engine=engine)
    assert [r.inner_it_A for r in rep1.records] == [r.inner_it_A for r in rep2.records]
    assert [r.scaled_res for r in rep1.records] == [r.scaled_res for r in rep2.records]


def test_c2_device_driver_matches_oracle():
    sol, rep, state = _gpu_run("c2")
    _check_against_golden(rep, "c2")
    _x_parity("c2", sol)


@pytest.mark.parametrize("name", ["c3s", "c5s"])
def test_reduced_configs_match_oracle(name):
    """Generalised pencils (config 3 family, mass matrices on both sides) and
    the 3-D r=4 config-5 family at reduced size."""
    sol, rep, state = _gpu_run(name)
    _check_against_golden(rep, name)
    _x_parity(name, sol)


def test_chunked_factor_download_matches_concat(monkeypatch, rng):
    """LowRankSolution._stack (adi.py:529-530 layout: Z = [z_1 ... z_k]): the
    double-buffered chunked download of large factors equals the one-copy path,
    for real and complex blocks and a ragged last chunk."""
    import torch
    from paper_2312_02891_b200.adi import LowRankSolution
    rows, r, k = 1531, 3, 7
    for dt in (torch.complex128, torch.float64):
        blocks = [torch.randn(rows, r, dtype=dt, device="cuda") for _ in range(k)]
        want = np.hstack([b.cpu().numpy().astype(complex) for b in blocks])
        monkeypatch.setattr(LowRankSolution, "CONCAT_BYTES", 1 << 40)
        assert np.array_equal(LowRankSolution._stack(blocks, rows, r), want)
        monkeypatch.setattr(LowRankSolution, "CONCAT_BYTES", 0)
        monkeypatch.setattr(LowRankSolution, "STAGE_BYTES", 200 * k * r * 16)   # 8 chunks
        monkeypatch.setattr(LowRankSolution, "_STAGING", None)
        got = LowRankSolution._stack(blocks, rows, r)
        assert got.shape == want.shape and np.array_equal(got, want)


def test_c3_intermediate_size_hard_shifts_match_oracle():
    """Config 3 at 250^2 / 175^2 with the full-size problem's pinned shifts, 8
    outer steps: at the small pair alpha ~ -1535, beta ~ -1575 the
    A-side Jacobi-GMRES(40) needs ~200 iterations per column on the CPU oracle
    too (75 at the other pairs) -- the stagnation seen at full size (1000 =
    max_inner_iterations on every column) is the algorithm's, not the device's.
    Per-step counts within +-2 per column (the records hold the sum over the
    three columns: +-6), tolerances to 1e-6, X parity to 1e-8."""
    sol, rep, state = _gpu_run("c3m")
    gold = read_steps_csv(os.path.join(GOLD, "oracle_c3m_gmres.csv"))
    assert rep.outer_iterations == len(gold) == 8
    hard = [g["inner_it_A"] for g in gold[1::2]]
    easy = [g["inner_it_A"] for g in gold[0::2]]
    assert min(hard) > 4 * max(easy)          # the oracle itself: the hard regime
    for rec, gd in zip(rep.records, gold):
        assert abs(rec.inner_it_A - gd["inner_it_A"]) <= 6, (rec.step, rec.inner_it_A, gd["inner_it_A"])
        assert abs(rec.inner_it_B - gd["inner_it_B"]) <= 6, (rec.step, rec.inner_it_B, gd["inner_it_B"])
        assert abs(rec.delta_A - gd["delta_A"]) <= 1e-6 * gd["delta_A"]
        assert abs(rec.scaled_res - gd["scaled_res"]) <= 1e-6 * gd["scaled_res"]
    _x_parity("c3m", sol)
