#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200 inner-solve hot path.

Default workload (BASELINE.json configs[1], "config 2"): inexact low-rank ADI
on the 3-D convection-diffusion pair n=64,000 / m=27,000, r=2, complex128,
pinned reference heuristic shifts (npairs=12), Jacobi-FGMRES(30) inner solves
with the paper's dynamic inner tolerance (dynamic_mid_bl), outer tolerance
1e-8.  One "step" = one full ADI solve to the 1e-8 residual.

  metric  = "wall time to 1e-8 ADI residual" (s, lower is better)
  value   = device-resident solve, inputs already in HBM
  e2e     = the public API call run(problem, config, shifts) with host
            scipy/numpy inputs: uploads, solve and the Z/Y download inside
  roofline= the dominant kernel class, from a CUDA-event-instrumented pass
  cpu_baseline = the reference's own CPU path (Jacobi-BiCGstab ADI, restated
            in oracle/) on the host, rank 0, N=1

`--impl reference` times that CPU path alone (the reference arm).
`--config c4` runs the inner-solve microbenchmark (SpMM/orthogonalisation GB/s).
Multi-GPU (torchrun): config 2 is single-GPU in BASELINE.json, so N ranks run
N independent replicas ("replicas only", weak scaling); value = max over ranks.
Configs 3/5 at N GPUs: A side on ranks [0, N/2), B side on [N/2, N), a side on
several GPUs row-partitioned (NCCL halo exchange + all-reduce); config 4 at N
GPUs: the operator row-partitioned over all N (strong scaling).  `--rowpart`
forces the row-partitioned path at N = 1.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
import warnings

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
if "--impl" in sys.argv and "reference" in sys.argv:
    # the reference's CPU path is scalar numpy/scipy: pin BLAS to one thread
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(_v, "1")

import numpy as np  # noqa: E402

PEAKS_FILE = os.path.join(REPO, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        with open(PEAKS_FILE) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


TRAFFIC_FILE = os.path.join(REPO, "profiles", "traffic.json")


def ncu_traffic(key):
    """DRAM bytes per launch of a kernel from a committed ncu capture
    (profiles/traffic.json, written by tools/ncu_traffic.py), or None."""
    try:
        with open(TRAFFIC_FILE) as fh:
            ent = json.load(fh)[key]
        return float(ent["traffic_bytes_per_launch"]), ent
    except Exception:
        return None, None


# -- distributed plumbing --------------------------------------------------------

class Dist:
    def __init__(self, want_gpus, force_pg=False):
        self.rank = int(os.environ.get("RANK", 0))
        self.world = int(os.environ.get("WORLD_SIZE", 1))
        self.local = int(os.environ.get("LOCAL_RANK", 0))
        self.pg = None
        if self.world > 1 or force_pg:
            import torch
            import torch.distributed as dist
            if self.world == 1:
                # a one-rank process group without torchrun (row-partitioned
                # path at N = 1)
                import socket
                with socket.socket() as sk:
                    sk.bind(("127.0.0.1", 0))
                    port = sk.getsockname()[1]
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", str(port))
                os.environ.setdefault("RANK", "0")
                os.environ.setdefault("WORLD_SIZE", "1")
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x):
        if not self.pg:
            return x
        import torch
        t = torch.tensor([float(x)], device="cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# -- clocks during the timed region ------------------------------------------------

class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region.

    Default: NVML queried in-process from a sampler thread (two light queries
    per sample; an nvidia-smi query takes the driver lock and stalled config-2
    steps by 20-50 ms).  SAD_CLOCKS=smi uses the recipe's nvidia-smi -lms loop."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device, period_ms=None):
        self.device = device
        self.mode = os.environ.get("SAD_CLOCKS", "nvml")
        self.period_ms = period_ms or (200 if self.mode == "nvml" else 1000)
        self.proc = None
        self.thread = None
        self.lines = []
        self.samples = []          # (sm_mhz, sm_max_mhz, set(reasons))
        self._stop = threading.Event()

    def start(self):
        if self.mode == "nvml":
            try:
                import pynvml
                pynvml.nvmlInit()
                idx = self.device
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                if vis:
                    idx = int(vis.split(",")[self.device])
                self._h = pynvml.nvmlDeviceGetHandleByIndex(idx)
                self._nv = pynvml
                self.thread = threading.Thread(target=self._poll, daemon=True)
                self.thread.start()
                return
            except Exception:
                self.mode = "smi"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self._nv, self._h
        bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
                "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(smax),
                                     {k for k, b in bits.items() if mask & b}))
            except Exception:
                pass
            self._stop.wait(self.period_ms / 1000.0)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.mode == "nvml" and self.thread is not None:
            self._stop.set()
            self.thread.join(timeout=2)
            sm = [x[0] for x in self.samples]
            reasons = set().union(*[x[2] for x in self.samples]) if self.samples else set()
            smax = self.samples[-1][1] if self.samples else None
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                    "reasons": sorted(reasons), "samples": len(sm), "source": "nvml"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


# -- workloads ------------------------------------------------------------------------

WORKLOADS = {
    "c2": "config 2: ADI to 1e-8, 3-D conv-diff 40^3/30^3, r=2, complex128, "
          "Jacobi-FGMRES(30), dynamic_mid_bl",
    "c3": "config 3: ADI to 1e-8, generalised 2-D Q1-FEM pencils 1000^2/700^2 (A+sM, B+sC), "
          "r=3, complex128, Jacobi-GMRES(40), dynamic_mid_bl",
    "c5": "config 5: ADI to 1e-8, 3-D conv-diff 200^3/160^3 (n=8M, m=4.1M), r=4, complex128, "
          "Jacobi-GMRES(30), dynamic_mid_bl, shifts generated on the GPU (device Ritz values)",
}
#: inner-iteration cap per column of the bounded CPU sample (first outer step)
CPU_SAMPLE_CAP = {"c3": 10, "c5": 1}


def build_c2(name="c2"):
    import paper_2312_02891_b200 as pb
    from paper_2312_02891_b200 import configs as cfgs
    spec = cfgs.CONFIGS[name]
    A, B, M, C, f, g = cfgs.build_problem(name)
    pairs, cyclic = spec.load_shift_pairs()
    prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
    cfg = pb.AdiConfig(strategy=spec.strategy, kmax=spec.kmax,
                       outer_tolerance=spec.outer_tolerance,
                       precond_kind_A="jacobi", precond_kind_B="jacobi")
    seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
    return spec, prob, cfg, seq, (A, B, M, C, f, g, pairs, cyclic)


def c2_config_json(spec, prob, extra=None):
    out = {"workload": WORKLOADS.get(spec.name, f"reduced {spec.name}"),
           "n": prob.n, "m": prob.m, "r": prob.r, "nnz_A": int(prob.A.nnz),
           "nnz_B": int(prob.B.nnz), "kmax": spec.kmax, "restart": spec.restart,
           "flexible": spec.flexible, "strategy": spec.strategy,
           "shifts": f"configs/shifts_{spec.name}.json (reference heuristic_shifts, "
                     f"npairs={spec.npairs})",
           "seed": spec.seed, "l2": "flushed between timed steps (256 MiB write)",
           "parallelism": "replicas"}
    if extra:
        out.update(extra)
    return out


def cpu_reference_solve(kmax=None):
    """The reference's own CPU path for config 2 (Jacobi-BiCGstab ADI), restated
    in oracle/ (the reference cannot travel to the GPU box).  Returns seconds
    and the outer step count."""
    from oracle import sylvadi_oracle as orc
    from paper_2312_02891_b200 import configs as cfgs
    spec = cfgs.CONFIGS["c2"]
    A, B, M, C, f, g = cfgs.build_problem("c2")
    pairs, cyclic = spec.load_shift_pairs()
    cfg = orc.Config(strategy=spec.strategy, kmax=kmax or spec.kmax,
                     outer_tolerance=spec.outer_tolerance)
    bA = orc.Binding("A", A, None, solver="bicgstab")
    bB = orc.Binding("B", B, None, solver="bicgstab")
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        run = orc.run_adi(A, B, f, g, cfg, pairs, bA, bB, cyclic=cyclic)
    return time.perf_counter() - t0, run.outer_iterations, bool(run.converged)


def cpu_reference_sample(name, max_inner):
    """Bounded CPU sample for configs 3/5 (a full reference solve would take
    hours on one core): the first outer step of the reference's Jacobi-BiCGstab
    ADI (oracle/ restatement) with the inner iterations capped per column."""
    from oracle import sylvadi_oracle as orc
    from paper_2312_02891_b200 import configs as cfgs
    spec = cfgs.CONFIGS[name]
    A, B, M, C, f, g = cfgs.build_problem(name)
    pairs, cyclic = spec.load_shift_pairs()
    cfg = orc.Config(strategy=spec.strategy, kmax=1, outer_tolerance=spec.outer_tolerance)
    bA = orc.Binding("A", A, M, solver="bicgstab", max_iterations=max_inner)
    bB = orc.Binding("B", B, C, solver="bicgstab", max_iterations=max_inner)
    from threadpoolctl import threadpool_limits
    t0 = time.perf_counter()
    with warnings.catch_warnings(), threadpool_limits(1):
        warnings.simplefilter("ignore")
        run = orc.run_adi(A, B, f, g, cfg, pairs, bA, bB, M=M, C=C, cyclic=cyclic)
    secs = time.perf_counter() - t0
    its = run.records[0].inner_it_A + run.records[0].inner_it_B if run.records else 0
    return secs, its


def run_reference_arm(args, dist):
    """--impl reference: rank 0 times the reference's CPU path (Jacobi-BiCGstab
    ADI, restated in oracle/) on the host, one full config-2 solve per step,
    sequentially in this process; other ranks exit without work."""
    if dist.rank != 0:
        return None
    for _ in range(args.warmup):
        cpu_reference_solve(kmax=1)
    secs, steps_cpu, conv = [], 0, True
    t0 = time.perf_counter()
    for _ in range(args.steps):
        t, steps_cpu, c = cpu_reference_solve()
        secs.append(t)
        conv = conv and c
    wall = time.perf_counter() - t0
    value = statistics.mean(secs)
    spec, prob, _, _, _ = build_c2()
    return {
        "metric": "wall time to 1e-8 ADI residual", "value": value, "unit": "s",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * value, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded reference generators)",
        "config": c2_config_json(spec, prob, {"outer_steps": steps_cpu, "converged": conv,
                                              "inner": "Jacobi-BiCGstab (reference path)"}),
        "cpu_baseline": {"value": value, "unit": "s", "cores": 1, "kind": "port",
                         "sample": f"{args.steps} full config-2 solves of the reference's "
                                   f"Jacobi-BiCGstab ADI (oracle/ restatement), sequential, "
                                   f"one core (BLAS threads 1); wall {wall:.1f}s"},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def profile_pass(eng):
    """One instrumented solve (CUDA events around every persistent launch,
    phase times from the kernel's %globaltimer).  Returns the 8 counters of
    sad_gmres_profile summed over both sides."""
    wss = list(eng.bA._workspaces.values()) + list(eng.bB._workspaces.values())
    for ws in wss:
        ws.profile(True)
    sol, rep, _ = eng.run()
    tot = np.zeros(13)
    for ws in wss:
        tot += ws.profile(False)
    return tot, rep


def run_ours_c2(args, dist, name="c2"):
    import torch
    import paper_2312_02891_b200 as pb
    from paper_2312_02891_b200 import _lib
    dev = dist.local
    torch.cuda.set_device(dev)
    lib = _lib.load()
    spec, prob, cfg, seq, raw = build_c2(name)
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible, device=dev)
    eng.warm()
    # the clock sampler starts before the warm-up: nvidia-smi's start-up (NVML
    # initialisation) stalls CUDA calls of this process for tens of ms
    clocks = Clocks(dev)
    clocks.start()
    # the L2-flush buffer is allocated and written once before the warm-up, and
    # every warm-up step follows the timed steps' flush-then-solve pattern
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        flush.fill_(1.0)
        _, rep, _ = eng.run()
    times, reps = [], []
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.sad_kernel_launches()
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _, rep, _ = eng.run()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        reps.append(rep)
    torch.cuda.synchronize()
    dist.barrier()
    ck = clocks.stop()
    launches = lib.sad_kernel_launches() - launches0
    ms = statistics.mean(times)
    ms_max = dist.max(ms)
    rep = reps[-1]
    step_ms = [round(x, 2) for x in times]

    # the same ADI with the reference's own inner algorithm on the device
    # (Jacobi-BiCGstab, solver="bicgstab"): the apples-to-apples comparison
    # with the reference arm's CPU BiCGstab
    same_alg = None
    if name == "c2":
        beng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                            device=dev, solver="bicgstab")
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            beng.run()
            torch.cuda.synchronize()
            bt = []
            for _ in range(2):
                flush.fill_(1.0)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                _, brep, _ = beng.run()
                e1.record()
                torch.cuda.synchronize()
                bt.append(e0.elapsed_time(e1))
        same_alg = {"solver": "Jacobi-BiCGstab with drift-resume (krylov.py:82-184) on the "
                              "device (sad_bicg_solve), batched over the r columns",
                    "value": statistics.mean(bt) / 1000.0, "unit": "s",
                    "outer_steps": brep.outer_iterations, "converged": brep.converged,
                    "sum_inner_A": brep.sum_inner_A, "sum_inner_B": brep.sum_inner_B}
        del beng
    # instrumented pass for the roofline: the dominant kernel is the persistent
    # GMRES kernel (one cooperative launch per inner solve)
    prof, prep = profile_pass(eng)
    peak, peak_kind = hbm_peak()
    kern_ms, kern_launches, kern_bytes = prof[0], prof[1], prof[2]
    ach = kern_bytes / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else 0.0
    traffic, tr_ent = ncu_traffic(f"{name}_persistent")
    if name in ("c3", "c5"):
        from paper_2312_02891_b200.verify import true_residual_norm
        sol, _, _ = eng.run()
        trn = true_residual_norm(prob, sol)
        del sol
    ab_mode = "concurrent" if eng.concurrent else "sequential"
    # large configs: free the timed engine before the e2e runs build their own
    if name in ("c3", "c5"):
        del eng
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        eng = None
    # e2e through the public API with host inputs
    e2e_times, e2e_solve = [], []
    A, B, M, C, f, g, pairs, cyclic = raw
    Zh = Yh = None
    for i in range(args.warmup + args.steps):
        Zh = Yh = None      # the previous step's factors are released first
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hprob = pb.SylvesterProblem(A=A, B=B, f=f, g=g, M=M, C=C)
        sol, erep = pb.run(hprob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                           device=dev)
        t1 = time.perf_counter()
        Zh, Yh = sol.Z, sol.Y
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_times.append(dt)
            e2e_solve.append(dict(erep.device_timing))
    e2e = dist.max(statistics.mean(e2e_times))
    def csr_bytes(X):
        return 0 if X is None else X.indptr.nbytes + X.indices.nbytes + X.data.nbytes
    h2d = csr_bytes(A) + csr_bytes(M) + 2 * (csr_bytes(B) + csr_bytes(C)) + f.nbytes + g.nbytes
    d2h = Zh.nbytes + Yh.nbytes

    line = {
        "metric": "wall time to 1e-8 ADI residual", "value": ms_max / 1000.0, "unit": "s",
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded reference generators)",
        "config": c2_config_json(spec, prob, {
            "outer_steps": rep.outer_iterations, "converged": rep.converged,
            "final_scaled_residual": rep.final_scaled_residual,
            "sum_inner_A": rep.sum_inner_A, "sum_inner_B": rep.sum_inner_B,
            "inner": f"Jacobi-{'F' if spec.flexible else ''}GMRES({spec.restart}) batched per "
                     f"column, delayed-Gram CGS2, device Givens",
            "ab_solves": ab_mode}),
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "traffic": traffic, "kernel": "k_gmres_persistent",
                     "traffic_source": tr_ent and (f"profiles/traffic.json[{name}_persistent]: "
                                                   f"{tr_ent['launches']} launches, "
                                                   f"{tr_ent['note']}"),
                     "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": kern_bytes / max(kern_launches, 1),
                     "avg_launch_ms": kern_ms / max(kern_launches, 1),
                     "measured": "CUDA events around each cooperative launch on its solve "
                                 "stream, instrumented pass over one full solve after the "
                                 "timed region"},
        "kernels": {"k_gmres_persistent": {"ms": kern_ms, "launches": int(kern_launches),
                                           "gbs": ach, "arnoldi_steps": int(prof[4]),
                                           "phaseA_ms(spmm+dots)": prof[3],
                                           "phaseC_ms(update)": prof[5],
                                           "cycle_end_ms": prof[6], "cycles": int(prof[7])},
                    "instrumented_solve_ms": prep.wall_ms},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "phases_ms": {k: statistics.mean(d.get(k, 0.0) for d in e2e_solve)
                              for k in ("construct_ms", "run_ms", "download_ms")},
                "step_s": [round(x, 4) for x in e2e_times],
                "step_phases_ms": [{k: round(d.get(k, 0.0), 1) for k in
                                    ("construct_ms", "run_ms", "download_ms")} for d in e2e_solve]},
        "gpu_launches": int(launches),
        "clocks": ck,
        "step_ms": step_ms,
    }
    if same_alg is not None:
        line["same_algorithm_as_reference"] = same_alg
    if name in ("c3", "c5"):
        line["config"]["true_scaled_residual"] = trn / rep.rhs_norm
        line["config"]["true_residual"] = "GPU power iteration (verify.true_residual_norm)"
    if name in CPU_SAMPLE_CAP and dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        cap = CPU_SAMPLE_CAP[name]
        secs, its = cpu_reference_sample(name, cap)
        line["cpu_baseline"] = {"value": secs, "unit": "s", "cores": 1, "kind": "port",
                                "sample": f"NOT a full solve: first outer step of the "
                                          f"reference's Jacobi-BiCGstab ADI (oracle/ "
                                          f"restatement) with inner iterations capped at {cap} "
                                          f"per column ({its} inner iterations in total)"}
    elif dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        secs, steps_cpu, conv = cpu_reference_solve()
        line["cpu_baseline"] = {"value": secs, "unit": "s", "cores": 1, "kind": "port",
                                "sample": f"one full config-2 solve of the reference's "
                                          f"Jacobi-BiCGstab ADI (oracle/ restatement), "
                                          f"{steps_cpu} outer steps, converged={conv}"}
    return line if dist.rank == 0 else None


def run_ours_c4(args, dist):
    """Inner-solve microbenchmark (config 4): shifted SpMM GB/s on the r=8 block
    (metric), plus 100 fixed GMRES steps through the persistent engine."""
    import torch
    from paper_2312_02891_b200 import GpuGmresBinding, _lib
    from paper_2312_02891_b200 import configs as cfgs
    dev = dist.local
    torch.cuda.set_device(dev)
    lib = _lib.load()
    n0 = args.c4_n0
    A, X = cfgs.build_c4(n0=n0, r=8, seed=0)
    # alpha = 0.1 * lambda_max estimate (Gershgorin bound of the stencil, negative)
    shift = 0.1 * (-abs(A.diagonal()).max() * 2.0)
    steps = args.c4_steps
    gb = GpuGmresBinding("A", A, None, precond_kind="jacobi", restart=steps, device=dev)
    rhs = torch.from_numpy(X).cuda()
    x = torch.empty_like(rhs)
    res = torch.empty_like(rhs)
    op = gb.operator(shift)
    n, r = A.shape[0], 8
    blk = n * r * 8
    spmm_b = A.nnz * 12 + 4 * (n + 1) + 2 * blk
    # --- shifted SpMM (the metric): K timed launches, L2 flushed in between ---
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    y = torch.empty_like(rhs)
    clocks = Clocks(dev)
    clocks.start()          # before the warm-up (see run_ours_c2)
    for _ in range(args.warmup):
        op.apply(rhs, y)
    time.sleep(0.3)         # the sampler's start-up is over before the timed region
    dist.barrier()
    torch.cuda.synchronize()
    l0 = lib.sad_kernel_launches()
    ms = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        op.apply(rhs, y)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    dist.barrier()
    launches = lib.sad_kernel_launches() - l0
    spmm_ms = statistics.mean(ms)
    spmm_gbs = spmm_b / (spmm_ms * 1e-3) / 1e9
    value = spmm_gbs * dist.world
    # --- the inner solve: 100 fixed GMRES steps, one persistent launch ---
    ws = gb.workspace(8, _lib.SAD_F64)
    ws.fixed(op, rhs, x, res, steps)
    _, tm = ws.fixed(op, rhs, x, res, steps, timed=True)
    ck = clocks.stop()
    peak, peak_kind = hbm_peak()
    solve_gbs = tm[3] / (tm[0] * 1e-3) / 1e9
    traffic, tr_ent = ncu_traffic("c4_spmm")
    straffic, str_ent = ncu_traffic("c4_persistent")
    line = {"metric": "inner SpMM GB/s", "value": value, "unit": "GB/s",
            "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": spmm_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"config 4: {n0}^2 conv-diff, r=8, "
                                                        f"shifted SpMM + {steps} fixed GMRES steps",
                                            "n": n, "nnz": int(A.nnz),
                                            "l2": "flushed between timed SpMMs"},
            "roofline": {"bound": "hbm", "achieved": spmm_gbs, "peak": peak, "unit": "GB/s",
                         "frac": spmm_gbs / peak, "traffic": traffic, "kernel": "k_spmm_bulk",
                         "traffic_source": tr_ent and (f"profiles/traffic.json[c4_spmm]: "
                                                       f"{tr_ent['note']}"),
                         "peak_kind": peak_kind, "algorithmic_bytes_per_launch": spmm_b},
            "inner_solve": {"kernel": "k_gmres_persistent", "steps": steps,
                            "kernel_ms": tm[0], "phaseA_ms": tm[1], "phaseC_ms": tm[2],
                            "algorithmic_bytes": tm[3], "gbs": solve_gbs,
                            "traffic": straffic,
                            "frac": solve_gbs / peak,
                            "iterations_per_s": steps * r / (tm[0] * 1e-3)},
            "gpu_launches": int(launches), "clocks": ck}
    return line if dist.rank == 0 else None


def run_ours_sharded(args, dist, name):
    """Configs 3/5 on N GPUs (one process per GPU): A side on ranks [0, N/2),
    B side on [N/2, N) (multigpu.ShardedAdi); a side on several GPUs is
    row-partitioned with NCCL halo exchange + all-reduce, a side on one GPU
    runs the persistent engine.  value = wall time to 1e-8 (max over ranks,
    total work fixed: strong scaling)."""
    import torch
    from paper_2312_02891_b200 import _lib
    from paper_2312_02891_b200.multigpu import make_sharded, side_groups
    dev = dist.local
    torch.cuda.set_device(dev)
    lib = _lib.load()
    spec, prob, cfg, seq, raw = build_c2(name)
    run = make_sharded(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                       device=dev, force_rowpart=args.rowpart)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        clocks = Clocks(dev)
        clocks.start()      # before the warm-up (see run_ours_c2)
        for _ in range(args.warmup):
            run.run()
        flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
        times = []
        dist.barrier()
        torch.cuda.synchronize()
        l0 = lib.sad_kernel_launches()
        for _ in range(args.steps):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            factors, gammas, rep = run.run()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            del factors
        torch.cuda.synchronize()
        dist.barrier()
        ck = clocks.stop()
    launches = lib.sad_kernel_launches() - l0
    ms_max = dist.max(statistics.mean(times))
    a_ranks, b_ranks = side_groups(dist.world)
    how = lambda rk: (f"row-partitioned over {len(rk)} GPUs (NCCL halo + all-reduce)"
                      if len(rk) > 1 or args.rowpart else "persistent engine on one GPU")
    line = {
        "metric": "wall time to 1e-8 ADI residual", "value": ms_max / 1000.0, "unit": "s",
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded reference generators)",
        "config": c2_config_json(spec, prob, {
            "outer_steps": rep.outer_iterations, "converged": rep.converged,
            "final_scaled_residual": rep.final_scaled_residual,
            "sum_inner_A": rep.sum_inner_A, "sum_inner_B": rep.sum_inner_B,
            "parallelism": f"A side on ranks {a_ranks}: {how(a_ranks)}; B side on ranks "
                           f"{b_ranks}: {how(b_ranks)}; one all_gather of partial Grams "
                           f"per outer step"}),
        "gpu_launches": int(launches), "clocks": ck,
    }
    return line if dist.rank == 0 else None


def run_ours_c4_rowpart(args, dist):
    """Config 4 under row partition (N GPUs, or N = 1 with --rowpart): the
    shifted SpMM with its halo exchange on every rank's slab, and the fixed
    GMRES steps through the row-partitioned engine (halo + all-reduce per
    reduction).  value = aggregate SpMM GB/s = global algorithmic bytes / max
    over ranks of the per-launch time (strong scaling: the matrix is fixed)."""
    import torch
    from paper_2312_02891_b200 import _lib
    from paper_2312_02891_b200 import configs as cfgs
    from paper_2312_02891_b200.rowpart import RowPartitionedGmres, _ptrs
    from paper_2312_02891_b200.device import current_stream_handle
    dev = dist.local
    torch.cuda.set_device(dev)
    lib = _lib.load()
    n0, steps = args.c4_n0, args.c4_steps
    A, X = cfgs.build_c4(n0=n0, r=8, seed=0)
    shift = 0.1 * (-abs(A.diagonal()).max() * 2.0)
    n, r = A.shape[0], 8
    rp = RowPartitionedGmres("A", A, None, precond_kind="jacobi", restart=steps,
                             max_iterations=steps, nranks=dist.world, comm="nccl", device=dev)
    pl = rp.plans[0]
    ops = rp.operator(shift)
    xl = torch.from_numpy(np.ascontiguousarray(X[pl.r0:pl.r1])).cuda()
    xe = torch.zeros((pl.n_loc + pl.n_halo, r), dtype=torch.float64, device="cuda")
    xe[:pl.n_loc] = xl
    y = torch.empty_like(xl)
    blk = n * r * 8
    spmm_b = A.nnz * 12 + 4 * (n + 1) + 2 * blk        # global algorithmic bytes
    halo_b = sum(p.n_halo for p in rp.all_plans) * r * 8

    def apply():
        rc = lib.sad_dist_op_apply(rp.comm.h, 1, _ptrs([ops[0].h]), _ptrs([rp._halos[0].h]), r,
                                   _lib.SAD_F64, _ptrs([xe.data_ptr()]), _ptrs([y.data_ptr()]),
                                   current_stream_handle())
        _lib.check(rc, rp._ctx)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    clocks = Clocks(dev)
    clocks.start()          # before the warm-up (see run_ours_c2)
    for _ in range(args.warmup):
        apply()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    l0 = lib.sad_kernel_launches()
    ms = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        apply()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    dist.barrier()
    launches = lib.sad_kernel_launches() - l0
    spmm_ms = dist.max(statistics.mean(ms))
    value = spmm_b / (spmm_ms * 1e-3) / 1e9
    # the fixed-step inner solve: `steps` Arnoldi steps (maxit = restart = steps)
    delta = 1e-300
    rp.solve_device(shift, xl, delta)          # warm
    torch.cuda.synchronize()
    dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    out = rp.solve_device(shift, xl, delta)
    e1.record()
    torch.cuda.synchronize()
    solve_ms = dist.max(e0.elapsed_time(e1))
    ck = clocks.stop()
    its = int(out.iterations[0])
    # DCGS2 (row-partitioned engine default): (2J + 2) N bytes per Arnoldi step j,
    # J = j + 1 (one dual dot sweep over V_0..V_j + w + v_j, one update sweep)
    N = blk
    orth_b = sum((2 * (j + 1) + 2) * N for j in range(its))
    spmm_arn = spmm_b + n * 8                    # + Jacobi gather
    solve_b = orth_b + its * spmm_arn + 2 * spmm_b
    peak, peak_kind = hbm_peak()
    line = {"metric": "inner SpMM GB/s", "value": value, "unit": "GB/s",
            "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": spmm_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config 4: {n0}^2 conv-diff, r=8, shifted SpMM + {steps} "
                                   f"GMRES steps, row-partitioned over {dist.world} GPU(s)",
                       "n": n, "nnz": int(A.nnz), "parallelism": f"row{dist.world}",
                       "halo_bytes_per_spmm": halo_b, "l2": "flushed between timed SpMMs"},
            "roofline": {"bound": "hbm", "achieved": value / dist.world, "peak": peak,
                         "unit": "GB/s", "frac": value / dist.world / peak, "traffic": None,
                         "kernel": "k_spmm (+ halo pack/exchange)", "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": spmm_b / dist.world},
            "inner_solve": {"engine": "row-partitioned multi-kernel DCGS2 (2 all-reduces/step)",
                            "steps": its,
                            "ms": solve_ms, "algorithmic_bytes": solve_b,
                            "gbs": solve_b / (solve_ms * 1e-3) / 1e9,
                            "frac_per_gpu": solve_b / (solve_ms * 1e-3) / 1e9 / dist.world / peak,
                            "iterations_per_s": its * r / (solve_ms * 1e-3)},
            "gpu_launches": int(launches), "clocks": ck}
    return line if dist.rank == 0 else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5", "c3s", "c5s"])
    ap.add_argument("--c4-n0", type=int, default=4096)
    ap.add_argument("--c4-steps", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rowpart", action="store_true",
                    help="configs 3-5: row-partitioned path even at N = 1 (NCCL world of 1)")
    args = ap.parse_args()
    if args.impl == "reference":
        dist = Dist(0)
        line = run_reference_arm(args, dist)
    else:
        sharded = args.config in ("c3", "c4", "c5", "c3s", "c5s") and (
            args.rowpart or int(os.environ.get("WORLD_SIZE", 1)) > 1)
        dist = Dist(args.gpus, force_pg=sharded)
        if args.config == "c4":
            line = run_ours_c4_rowpart(args, dist) if sharded else run_ours_c4(args, dist)
        elif sharded:
            line = run_ours_sharded(args, dist, args.config)
        else:
            line = run_ours_c2(args, dist, args.config)
    if line is not None:
        print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
