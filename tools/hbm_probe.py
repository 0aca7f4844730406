"""HBM read / write / copy bandwidth of the box (torch ops, CUDA events): compares boxes."""
import torch
n = 1 << 30  # 1 Gi fp32 = 4 GiB
x = torch.empty(n, dtype=torch.float32, device="cuda")
y = torch.empty(n, dtype=torch.float32, device="cuda")
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3
w = t(lambda: x.fill_(1.0)); print(f"write {4 * n / w / 1e9:.0f} GB/s")
r = t(lambda: x.sum()); print(f"read {4 * n / r / 1e9:.0f} GB/s")
c = t(lambda: y.copy_(x)); print(f"copy {8 * n / c / 1e9:.0f} GB/s (read+write)")
