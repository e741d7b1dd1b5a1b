#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200 inner-solve hot path.

Default workload (BASELINE.json configs[3], "config 4", the configuration the
metric "inner SpMM GB/s vs HBM peak" is quoted on): the shifted SpMM
y = (A + alpha I) x of the inner solves on a 2-D 5-point convection-diffusion
operator on a 4096^2 grid (16.7M rows, 84M nonzeros) and an r = 8 fp64 block.
One "step" = one shifted SpMM over the whole block.

  metric  = "inner SpMM GB/s" (algorithmic bytes / time, higher is better)
  value   = device-resident SpMM (k_spmm_bulk), CUDA events, L2 flushed
  e2e     = the same SpMM through the host-buffer C-ABI call
            (DeviceOperator.apply_host -> sad_op_apply_host): pinned host x in,
            host y out, transfers inside the timed region
  roofline= k_spmm_bulk against the measured HBM copy bandwidth
  inner_solve = 100 fixed Jacobi-GMRES steps in one persistent launch
            (orthogonalisation GB/s, iterations/s)
  config3_wall_time = config 3's 1-GPU wall time to the 1e-8 ADI residual
  cpu_baseline = the reference's ShiftedOperator.apply (oracle/ restatement)
            on all host threads, rank 0, N=1

`--impl reference` times that CPU apply alone (the reference arm).
`--config c2|c3|c5` times a whole ADI solve to 1e-8 (wall time, lower is
better; the reference arm then runs the reference's Jacobi-BiCGstab ADI).
Multi-GPU (torchrun): config 4 row-partitions the operator over the N ranks
(NCCL halo exchange; aggregate SpMM GB/s, strong scaling); configs 3/5 put the
A side on ranks [0, N/2) and the B side on [N/2, N), a side on several GPUs
row-partitioned; config 2 runs N replicas.  `--rowpart` forces the
row-partitioned path at N = 1.
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
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible, device=dev,
                       engine=args.engine)
    engine = eng.engine          # "auto" resolved: persistent, or the ring multi-kernel engine
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
    trn = None
    if name in ("c3", "c5"):
        from paper_2312_02891_b200.verify import true_residual_norm
        sol, _, _ = eng.run()
        trn = true_residual_norm(prob, sol)
        del sol
    ab_mode = "concurrent" if eng.concurrent else "sequential"

    def free_engine():
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        for ctx in list(_lib._CTX.values()):
            lib.sad_ctx_trim(ctx)

    if engine == "persistent":
        prof, prep = profile_pass(eng)
    else:
        # the multi-kernel engine has no byte counters: the algorithmic bytes of the
        # solve (same algorithm, same iteration counts) are counted by one
        # instrumented solve of the persistent engine, and divided by the TIMED
        # solve of the engine that ran (all its kernels, launch gaps included)
        del eng
        eng = None
        free_engine()
        peng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible,
                            device=dev, engine="persistent")
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            peng.run()
            prof, prep = profile_pass(peng)
        del peng
        assert prep.sum_inner_A == rep.sum_inner_A and prep.sum_inner_B == rep.sum_inner_B
        prof = prof.copy()
        prof[0] = ms
    peak, peak_kind = hbm_peak()
    kern_ms, kern_launches, kern_bytes = prof[0], prof[1], prof[2]
    ach = kern_bytes / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else 0.0
    traffic, tr_ent = ncu_traffic(f"{name}_persistent")
    # large configs: free the timed engine before the e2e runs build their own
    if name in ("c3", "c5"):
        eng = None
        free_engine()
    # e2e through the public API with host inputs
    e2e_times, e2e_solve = [], []
    A, B, M, C, f, g, pairs, cyclic = raw
    Zh = Yh = None
    sol = erep = None
    for i in range(args.warmup + args.steps):
        Zh = Yh = None      # the previous step's factors are released first
        sol = erep = None   # (host arrays and the device blocks behind them)
        if name in ("c3", "c5"):
            free_engine()
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
                     "frac": ach / peak, "traffic": traffic,
                     "kernel": "k_gmres_persistent" if engine == "persistent" else
                               "k_dot_dual_ring + k_update_ring + k_spmm_band (whole timed solve)",
                     "engine": engine,
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


C4_WORKLOAD = ("config 4: inner-solve microbenchmark, 2-D 5-point conv-diff 100*(1,1).grad on "
               "a {n0}^2 grid (n={n}, nnz={nnz}), shifted SpMM y = (A + alpha I) x on an "
               "r=8 fp64 Gaussian block, alpha = 0.1 * lambda_max (largest-magnitude Ritz "
               "value, {ritz} Arnoldi steps); plus {steps} fixed Jacobi-GMRES steps")


def c4_shift(A, dev, steps=10):
    """alpha = 0.1 * lambda_max estimate: the largest-magnitude Ritz
    value of `steps` Arnoldi iterations (shifts.arnoldi_ritz on the device,
    start vector ones as pencil_ritz_sets, shifts.py:111)."""
    from paper_2312_02891_b200.device import DeviceMatrix, DeviceOperator
    from paper_2312_02891_b200.shifts import arnoldi_ritz
    dm = DeviceMatrix(A, False, dev)
    op0 = DeviceOperator(dm, None, 0.0, precond_kind="none")
    ritz = arnoldi_ritz(lambda v: op0.apply(v), np.ones(A.shape[0]), steps, device=dev)
    lam = complex(ritz.values[np.argmax(np.abs(ritz.values))])
    del op0, dm
    return 0.1 * lam.real, lam


def c4_pinned_shift(n0):
    """configs/shift_c4.json (configs/make_shift_c4.py: the reference's own
    arnoldi_ritz), or None for another grid size."""
    try:
        with open(os.path.join(REPO, "configs", "shift_c4.json")) as fh:
            d = json.load(fh)
    except OSError:
        return None
    if int(d["n0"]) != int(n0):
        return None
    return float(d["shift"]), complex(*d["lambda_max"])


def c4_spmm_bytes(A, r=8, s=8):
    """Algorithmic bytes of one shifted SpMM: CSR (values, columns,
    row offsets) + read x + write y; no Jacobi gather in apply mode."""
    n = A.shape[0]
    return A.nnz * 12 + 4 * (n + 1) + 2 * s * r * n


def cpu_apply_threads(A, X, shift, threads, reps=1, out=None):
    """The reference's ShiftedOperator.apply (sparse.py:192-206) on the host:
    the oracle restatement (oracle/sylvadi_oracle.py ShiftedOp.apply: scipy
    csr_matvecs, cast to complex, + shift * x) over `threads` row chunks in
    parallel (scipy's sparsetools and numpy release the GIL).  Returns the
    seconds of each repetition and the output block."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import sylvadi_oracle as orc
    n = A.shape[0]
    nchunk = max(1, 4 * threads)
    bnd = np.linspace(0, n, nchunk + 1).astype(np.int64)
    ops = []
    for i in range(nchunk):
        r0, r1 = int(bnd[i]), int(bnd[i + 1])
        # the row slab as a square operator over the slab's rows needs the full
        # column range: apply the slab of A, then the shift on the slab's rows
        ops.append((A[r0:r1], r0, r1))
    if out is None:
        out = np.empty((n, X.shape[1]), dtype=np.complex128)

    def work(i):
        Ai, r0, r1 = ops[i]
        # orc.ShiftedOp(Ai, None, shift).apply would check squareness; the slab
        # form is the same arithmetic: (A x).astype(complex) + shift * x
        y = (Ai @ X).astype(complex)
        y += complex(shift) * X[r0:r1]
        out[r0:r1] = y

    assert orc.ShiftedOp is not None
    secs = []
    with ThreadPoolExecutor(threads) as ex:
        for _ in range(reps):
            t0 = time.perf_counter()
            list(ex.map(work, range(nchunk)))
            secs.append(time.perf_counter() - t0)
    return secs, out


def run_reference_arm_c4(args, dist):
    """--impl reference, config 4: the reference's CPU shifted SpMM
    (ShiftedOperator.apply, sparse.py:192-206, via the oracle restatement) on
    the full config-4 block, all host threads; one full apply per step."""
    if dist.rank != 0:
        return None
    from paper_2312_02891_b200 import configs as cfgs
    n0 = args.c4_n0
    A, X = cfgs.build_c4(n0=n0, r=8, seed=0)
    pinned = c4_pinned_shift(n0)
    if args.c4_shift is not None:
        shift = float(args.c4_shift)
    elif pinned is not None:
        shift = pinned[0]
    else:
        raise SystemExit("config 4 at this grid size needs --c4-shift (the pinned shift is for "
                         "the 4096^2 grid)")
    threads = len(os.sched_getaffinity(0))
    spmm_b = c4_spmm_bytes(A)
    cpu_apply_threads(A, X, shift, threads, reps=args.warmup)
    secs, _ = cpu_apply_threads(A, X, shift, threads, reps=args.steps)
    mean = statistics.mean(secs)
    value = spmm_b / mean / 1e9
    n = A.shape[0]
    return {
        "metric": "inner SpMM GB/s", "value": value, "unit": "GB/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * mean, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded reference generators)",
        "config": {"workload": C4_WORKLOAD.format(n0=n0, n=n, nnz=A.nnz, ritz="-", steps=0),
                   "n": n, "nnz": int(A.nnz), "r": 8, "shift": shift,
                   "algorithmic_bytes_per_step": spmm_b},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full config-4 applies (16.7M x 8 block) of the "
                                   f"reference's ShiftedOperator.apply (oracle/ restatement: "
                                   f"scipy csr_matvecs, complex cast, + shift x) over "
                                   f"{threads} threads on row chunks; the reference itself "
                                   f"is single-threaded"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def c3_wall_time(args, dev):
    """Config 3's 1-GPU wall time to the 1e-8 ADI residual (BASELINE configs[2]):
    the device-resident solve (one warm-up run, one timed run, CUDA events)."""
    import torch
    import paper_2312_02891_b200 as pb
    spec, prob, cfg, seq, _ = build_c2("c3")
    eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible, device=dev)
    eng.warm()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        eng.run()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _, rep, _ = eng.run()
        e1.record()
        torch.cuda.synchronize()
    secs = e0.elapsed_time(e1) / 1000.0
    out = {"workload": WORKLOADS["c3"], "value": secs, "unit": "s",
           "measured": "CUDA events around one device-resident solve after one warm-up solve",
           "outer_steps": rep.outer_iterations, "converged": rep.converged,
           "final_scaled_residual": rep.final_scaled_residual,
           "sum_inner_A": rep.sum_inner_A, "sum_inner_B": rep.sum_inner_B}
    del eng
    return out


def _free_device():
    import gc
    import torch
    from paper_2312_02891_b200 import _lib, krylov
    krylov._POOL.clear()          # pooled Krylov workspaces (config 4: 108 GB of basis)
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    lib = _lib.load()
    for ctx in list(_lib._CTX.values()):
        lib.sad_ctx_trim(ctx)


def run_ours_c4(args, dist):
    """Config 4 (BASELINE configs[3], the metric "inner SpMM GB/s vs HBM peak"):
    the shifted SpMM on the full 16.7M x 8 block (value: device-resident; e2e:
    host block -> sad_op_apply_host -> host block), then 100 fixed GMRES steps
    (orthogonalisation GB/s, iterations/s) and config 3's 1-GPU wall time."""
    import torch
    from paper_2312_02891_b200 import GpuGmresBinding, _lib
    from paper_2312_02891_b200 import configs as cfgs
    dev = dist.local
    torch.cuda.set_device(dev)
    lib = _lib.load()
    n0 = args.c4_n0
    A, X = cfgs.build_c4(n0=n0, r=8, seed=0)
    ritz_steps = 10
    pinned = c4_pinned_shift(n0)
    if args.c4_shift is not None:
        shift, lam = float(args.c4_shift), None
    elif pinned is not None:
        shift, lam = pinned          # configs/shift_c4.json (the reference's arnoldi_ritz)
    else:
        shift, lam = c4_shift(A, dev, ritz_steps)
    steps = args.c4_steps
    gb = GpuGmresBinding("A", A, None, precond_kind="jacobi", restart=steps, device=dev)
    rhs = torch.from_numpy(X).cuda()
    op = gb.operator(shift)
    n, r = A.shape[0], 8
    blk = n * r * 8
    spmm_b = c4_spmm_bytes(A)
    # --- shifted SpMM (the metric): K timed launches, L2 flushed in between ---
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    y = torch.empty_like(rhs)
    clocks = Clocks(dev)
    clocks.start()          # before the warm-up (see run_ours_c2)
    op.apply(rhs, y)        # builds the banded plan (host inspector, once per pattern)
    torch.cuda.synchronize()
    time.sleep(0.3)         # the sampler's start-up is over before the warm-up: the W
                            # warm-up steps run back to back with the timed ones (an idle
                            # gap right before the timed region costs the first launch 15 %)
    for _ in range(args.warmup):
        flush.fill_(1.0)
        op.apply(rhs, y)
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
    torch.cuda.synchronize()
    dist.barrier()
    launches = lib.sad_kernel_launches() - l0
    ck = clocks.stop()
    spmm_ms = dist.max(statistics.mean(ms))
    spmm_gbs = spmm_b / (spmm_ms * 1e-3) / 1e9
    value = spmm_gbs * dist.world
    y_dev = y.cpu().numpy()
    # --- e2e: the same SpMM through the host-buffer C-ABI call (pinned host
    # blocks; every step uploads x and downloads y inside the timed region) ---
    xh = torch.empty((n, r), dtype=torch.float64, pin_memory=True)
    yh = torch.empty((n, r), dtype=torch.float64, pin_memory=True)
    xh.copy_(torch.from_numpy(X))
    xh_np, yh_np = xh.numpy(), yh.numpy()
    for _ in range(args.warmup):
        op.apply_host(xh_np, yh_np)
    e2e_s = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op.apply_host(xh_np, yh_np)           # synchronous: y is on the host
        e2e_s.append(time.perf_counter() - t0)
    e2e_mean = dist.max(statistics.mean(e2e_s))
    e2e_gbs = spmm_b / e2e_mean / 1e9 * dist.world
    host_vs_dev = float(np.max(np.abs(yh_np - y_dev)))
    del xh, yh
    # --- the inner solve: 100 fixed GMRES steps, one persistent launch ---
    x = torch.empty_like(rhs)
    res = torch.empty_like(rhs)
    ws = gb.workspace(8, _lib.SAD_F64)
    ws.fixed(op, rhs, x, res, steps)
    _, tm = ws.fixed(op, rhs, x, res, steps, timed=True)
    peak, peak_kind = hbm_peak()
    solve_gbs = tm[3] / (tm[0] * 1e-3) / 1e9
    arn = int(tm[6]) if tm[6] > 0 else steps
    # DCGS2 bytes of Arnoldi step j (J = j + 1 basis blocks): (2J + 2) N
    orth_b = sum((2 * (j + 1) + 2) * blk for j in range(arn))
    orth_ms = max(tm[1] - tm[4], 0.0) + tm[2]
    band = op.band_info()
    spmm_kernel = "k_spmm_band" if band else "k_spmm_bulk"
    traffic, tr_ent = ncu_traffic("c4_spmm_band" if band else "c4_spmm")
    straffic, str_ent = ncu_traffic("c4_persistent")
    del gb, op, ws, x, res, y
    _free_device()
    # the same 100 steps through the ring multi-kernel engine (what DeviceAdi's
    # engine="auto" runs on blocks this large, and what every rank of a
    # row-partitioned run executes on its slab)
    ring = None
    try:
        from paper_2312_02891_b200.rowpart import RowPartitionedGmres
        rpg = RowPartitionedGmres("A", A, None, precond_kind="jacobi", restart=steps,
                                  max_iterations=steps, nranks=1, comm="local", device=dev)
        rpg.solve_device(shift, rhs, 1e-300)          # warm (plans, workspaces)
        torch.cuda.synchronize()
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        rout = rpg.solve_device(shift, rhs, 1e-300)
        e1.record()
        torch.cuda.synchronize()
        rms = e0.elapsed_time(e1)
        ring = {"engine": "multi-kernel delayed-Gram CGS2: k_spmm_band, k_dot_dual_ring, "
                          "k_update_ring, device finishers (csrc/sad_ring.cuh)",
                "steps": int(rout.iterations[0]), "ms": rms, "algorithmic_bytes": tm[3],
                "gbs": tm[3] / (rms * 1e-3) / 1e9, "frac": tm[3] / (rms * 1e-3) / 1e9 / peak,
                "measured": "CUDA events around the whole solve (all kernels, launch gaps included)"}
        del rpg, rout
    except Exception as exc:              # reported, never hidden
        ring = {"error": f"{type(exc).__name__}: {exc}"}
    del rhs, flush
    _free_device()
    c3 = None
    if not args.no_c3:
        try:
            c3 = c3_wall_time(args, dev)
        except Exception as exc:          # reported, never hidden
            c3 = {"error": f"{type(exc).__name__}: {exc}"}
        _free_device()
    line = {"metric": "inner SpMM GB/s", "value": value, "unit": "GB/s",
            "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": spmm_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded reference generators: convdiff_fd, Philox N(0,1))",
            "config": {"workload": C4_WORKLOAD.format(n0=n0, n=n, nnz=A.nnz, ritz=ritz_steps,
                                                      steps=steps),
                       "n": n, "nnz": int(A.nnz), "r": r, "shift": shift,
                       "lambda_max_ritz": None if lam is None else [lam.real, lam.imag],
                       "l2": "flushed between timed SpMMs (256 MiB write); the 3.36 GB "
                             "working set also exceeds L2",
                       "parallelism": "single GPU" if dist.world == 1 else "replicas"},
            "roofline": {"bound": "hbm", "achieved": spmm_gbs, "peak": peak, "unit": "GB/s",
                         "frac": spmm_gbs / peak, "traffic": traffic, "kernel": spmm_kernel,
                         "frac_of_nominal_8000": spmm_gbs / 8000.0,
                         # the banded plan stores 16-bit local columns and no row offsets:
                         # its DRAM traffic is below the CSR's algorithmic bytes, so the
                         # device's own rate is traffic / time
                         "dram_gbs": traffic / (spmm_ms * 1e-3) / 1e9 if traffic else None,
                         "dram_frac": traffic / (spmm_ms * 1e-3) / 1e9 / peak if traffic else None,
                         "band_plan": band,
                         "note": "frac = SURVEY 8d's algorithmic (CSR) bytes / time / peak; the banded "
                                 "plan moves fewer bytes than that formula (10 B per nonzero, no row "
                                 "offsets), so frac can pass 1.0 -- dram_frac (ncu DRAM traffic / time / "
                                 "peak) is the device's own rate" if band else None,
                         "traffic_source": tr_ent and (f"profiles/traffic.json[c4_spmm]: "
                                                       f"{tr_ent['note']}"),
                         "peak_kind": peak_kind, "algorithmic_bytes_per_launch": spmm_b,
                         "avg_launch_ms": spmm_ms,
                         "launch_ms": [round(t, 4) for t in ms],
                         "measured": "CUDA events around each timed launch on torch's current "
                                     "stream (the launch stream)"},
            "e2e": {"value": e2e_gbs, "unit": "GB/s", "h2d_bytes_per_step": blk,
                    "d2h_bytes_per_step": blk, "ms_per_step": e2e_mean * 1000.0,
                    "api": "DeviceOperator.apply_host -> sad_op_apply_host (pinned host x, y; "
                           "chunked upload / SpMM / download overlapped)",
                    "max_abs_diff_vs_device_apply": host_vs_dev},
            "inner_solve": {"kernel": "k_gmres_persistent", "steps": arn,
                            "kernel_ms": tm[0], "phaseA_ms": tm[1], "phaseC_ms": tm[2],
                            "spmm_subphase_ms": tm[4], "cycle_end_ms": tm[5],
                            "algorithmic_bytes": tm[3], "gbs": solve_gbs,
                            "frac": solve_gbs / peak, "traffic": straffic,
                            "orthogonalisation_bytes": orth_b,
                            "orthogonalisation_ms": orth_ms,
                            "orthogonalisation_gbs": orth_b / (orth_ms * 1e-3) / 1e9
                            if orth_ms > 0 else None,
                            "iterations_per_s": arn * r / (tm[0] * 1e-3),
                            "note": "phase times from block 0's %globaltimer; orthogonalisation "
                                    "= phase A minus its SpMM sub-phase, plus phase C"},
            "gpu_launches": int(launches), "clocks": ck}
    if ring is not None:
        line["inner_solve_ring_engine"] = ring
    if c3 is not None:
        line["config3_wall_time"] = c3
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        cpu_reps = 40          # ~10 s of wall time on 16 threads (the bounded CPU sample)
        secs, ycpu = cpu_apply_threads(A, X, shift, threads, reps=cpu_reps)
        t = statistics.mean(secs)
        rel = float(np.max(np.abs(ycpu - y_dev)) / np.max(np.abs(ycpu)))
        line["cpu_baseline"] = {"value": spmm_b / t / 1e9, "unit": "GB/s", "cores": threads,
                                "kind": "port",
                                "sample": f"{cpu_reps} full config-4 applies of the reference's "
                                          f"ShiftedOperator.apply (oracle/ restatement, scipy "
                                          f"csr_matvecs + complex cast + shift) over {threads} "
                                          f"threads on row chunks, {t:.2f} s each"}
        line["parity"] = {"max_rel_diff_vs_cpu_apply": rel,
                          "note": "device SpMM vs the reference's apply on the full block "
                                  "(fma vs mul+add rounding)"}
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
    pinned = c4_pinned_shift(n0)          # configs/shift_c4.json (the reference's arnoldi_ritz)
    shift = pinned[0] if pinned is not None else 0.1 * (-abs(A.diagonal()).max() * 2.0)
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
    ap.add_argument("--config", default="c4", choices=["c2", "c3", "c4", "c5", "c3s", "c5s"])
    ap.add_argument("--c4-n0", type=int, default=4096)
    ap.add_argument("--c4-steps", type=int, default=100)
    ap.add_argument("--c4-shift", type=float, default=None,
                    help="config 4 shift (default: 0.1 * largest-magnitude Ritz value)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3", action="store_true",
                    help="config 4: skip the config-3 wall-time key")
    ap.add_argument("--engine", default="auto", choices=["auto", "persistent", "rowpart"],
                    help="ADI configs: inner engine (auto: the ring multi-kernel engine for "
                         "large blocks, else one persistent launch per solve)")
    ap.add_argument("--rowpart", action="store_true",
                    help="configs 3-5: row-partitioned path even at N = 1 (NCCL world of 1)")
    args = ap.parse_args()
    if args.impl == "reference":
        dist = Dist(0)
        line = (run_reference_arm_c4(args, dist) if args.config == "c4"
                else run_reference_arm(args, dist))
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
