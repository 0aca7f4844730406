"""Run a few DisCo steps for ncu (no timing here; numbers under ncu are never bench values).

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python tools/profile_step.py
  ncu --set full --clock-control none --import-source on -k regex:"logits|gemm" -c 4 \
      -o gpurun_out/prof python tools/profile_step.py
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32768)
ap.add_argument("--dim", type=int, default=512)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
torch.cuda.set_device(0)
g = torch.Generator(device="cuda")
g.manual_seed(0)
I = torch.nn.functional.normalize(torch.randn(a.batch, a.dim, device="cuda", generator=g), dim=1).bfloat16()
T = torch.nn.functional.normalize(torch.randn(a.batch, a.dim, device="cuda", generator=g), dim=1).bfloat16()
for _ in range(a.steps):
    _, _, plan = P.disco_step_async(P.SingleEndpoint(), I, T, 100.0)
print("loss", P.finish_status(plan))
