"""Config 2 timed solve under different side conditions: L2 flush before each
step, nvidia-smi clock sampling (subprocess) and NVML sampling (in-process)."""
import os
import subprocess
import sys
import threading
import time
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_02891_b200 as pb  # noqa: E402
from paper_2312_02891_b200 import configs as cfgs  # noqa: E402

warnings.simplefilter("ignore")
spec = cfgs.CONFIGS["c2"]
A, B, M, C, f, g = cfgs.build_problem("c2")
pairs, cyclic = spec.load_shift_pairs()
prob = pb.SylvesterProblem(A=A, B=B, f=f, g=g)
cfg = pb.AdiConfig(strategy=spec.strategy, kmax=spec.kmax, precond_kind_A="jacobi",
                   precond_kind_B="jacobi")
seq = pb.ShiftSequence(pairs=pairs, cyclic=cyclic)
eng = pb.DeviceAdi(prob, cfg, seq, restart=spec.restart, flexible=spec.flexible)
eng.warm()
for _ in range(3):
    eng.run()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def timed(n=5, do_flush=False):
    ts = []
    for _ in range(n):
        if do_flush:
            flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sum(ts) / len(ts)


print("plain", timed())
print("flush", timed(do_flush=True))
FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
          "clocks_event_reasons.hw_thermal_slowdown,"
          "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
for period in (200, 1000):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={FIELDS}", "--format=csv,noheader,nounits",
                          "-lms", str(period)], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    time.sleep(0.5)
    print(f"nvidia-smi -lms {period}", timed(do_flush=True))
    p.terminate()
    p.wait()
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    stop = False
    samples = []

    def loop():
        while not stop:
            samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.2)
    th = threading.Thread(target=loop, daemon=True)
    th.start()
    print("nvml 200ms", timed(do_flush=True), "samples", len(samples))
    stop = True
    th.join()
except Exception as e:
    print("nvml", e)
