"""Bitwise check that an experiment flag setting leaves the step's outputs unchanged.

  python tools/flag_parity.py --flags 16384 [--batch 8192 --dim 512 --world 1]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402
from paper_2304_08480_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8192)
ap.add_argument("--dim", type=int, default=512)
ap.add_argument("--flags", type=int, nargs="+", required=True)
a = ap.parse_args()
torch.cuda.set_device(0)
g = torch.Generator(device="cuda")
g.manual_seed(0)
I = torch.nn.functional.normalize(torch.randn(a.batch, a.dim, device="cuda", generator=g), dim=1).bfloat16()
T = torch.nn.functional.normalize(torch.randn(a.batch, a.dim, device="cuda", generator=g), dim=1).bfloat16()


def run(flags):
    _lib.load().disco_b200_set_experiment_flags(flags)
    di, dt, loss = P.disco_step(None, I, T, 100.0)
    _lib.load().disco_b200_set_experiment_flags(0)
    return di.clone(), dt.clone(), loss


base = run(0)
for f in a.flags:
    got = run(f)
    same = torch.equal(base[0], got[0]) and torch.equal(base[1], got[1]) and base[2] == got[2]
    print(f"flags {f}: {'bitwise identical' if same else 'DIFFERENT'} (loss {got[2]!r})")
