"""e2e (host-buffer) step time of this checkout, for A/B against another checkout (separate processes).

  python tools/e2e_ab.py [--reps 12]      prints the median e2e step time in ms (bench's e2e recipe)
"""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32768)
ap.add_argument("--dim", type=int, default=512)
ap.add_argument("--reps", type=int, default=12)
ap.add_argument("--set", action="append", default=[],
                help="NAME=VALUE: set a module switch in paper_2304_08480_b200.shard (Python literal)")
a = ap.parse_args()
if a.set:
    import ast
    from paper_2304_08480_b200 import shard
    for kv in a.set:
        name, val = kv.split("=", 1)
        setattr(shard, name, ast.literal_eval(val))
torch.cuda.set_device(0)
g = torch.Generator(device="cuda")
g.manual_seed(1234)
I = torch.nn.functional.normalize(torch.randn(a.batch, a.dim, device="cuda", generator=g), dim=1).bfloat16()
T = torch.nn.functional.normalize(torch.randn(a.batch, a.dim, device="cuda", generator=g), dim=1).bfloat16()
I_h, T_h = I.cpu().pin_memory(), T.cpu().pin_memory()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(3):
    P.disco_step(None, I_h, T_h, 100.0)
ms = []
for _ in range(a.reps):
    flush.zero_()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    di, dt, loss = P.disco_step(None, I_h, T_h, 100.0)
    s1.record()
    s1.synchronize()
    ms.append(s0.elapsed_time(s1))
print(f"{' '.join(a.set) or 'default'}: e2e median {statistics.median(ms):.4f} ms min {min(ms):.4f} loss {loss:.6f}")
