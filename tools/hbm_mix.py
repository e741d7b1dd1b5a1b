"""HBM bandwidth of plain torch streaming kernels at several read:write mixes
(calibration for the SpMM's 2:1 mix; the driver's peak is a 1:1 copy)."""
import torch

n = 1 << 27                      # 1 GiB of fp64 per tensor
a = torch.rand(n, dtype=torch.float64, device="cuda")
b = torch.rand(n, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)


def best(fn, nbytes, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    t = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    return nbytes / (min(t) * 1e-3) / 1e9


print(f"copy 1:1    {best(lambda: c.copy_(a), 16 * n):8.0f} GB/s")
print(f"add  2:1    {best(lambda: torch.add(a, b, out=c), 24 * n):8.0f} GB/s")
print(f"sum  1:0    {best(lambda: a.sum(), 8 * n):8.0f} GB/s")
print(f"fill 0:1    {best(lambda: c.fill_(1.0), 8 * n):8.0f} GB/s")
