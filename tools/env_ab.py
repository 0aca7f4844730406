"""Single-rank path switches A/B: an environment switch (default DISCO_SYMMETRIC, the symmetric
forward; DISCO_HFUSE, the fused backward) at 1 against 0.

  python tools/env_ab.py [--var DISCO_SYMMETRIC] [--sizes 2048x512 8192x512 32768x512 16384x1024] [--reps 10]

For each size: both paths on the same device inputs, their normwise difference, the symmetric
path against the f64 oracle on sampled rows, and the device step time of each (CUDA events,
L2 flushed between steps).
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402
from oracle import disco_oracle as O  # noqa: E402
from paper_2304_08480_b200.shard import clear_plans  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", nargs="+", default=["2048x512", "8192x512", "32768x512", "16384x1024"])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--t", type=float, default=100.0)
ap.add_argument("--var", default="DISCO_SYMMETRIC")
a = ap.parse_args()
dev = torch.device("cuda", 0)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)


def run(I, T, sym, reps):
    os.environ[a.var] = "1" if sym else "0"
    clear_plans()
    out = P.disco_step(None, I, T, a.t)
    torch.cuda.synchronize()
    ms = []
    for i in range(reps + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.disco_step(None, I, T, a.t)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ms.append(e0.elapsed_time(e1))
    return out, statistics.median(ms)


res = {}
for sz in a.sizes:
    B, D = map(int, sz.split("x"))
    I, T = O.synthetic_features(B, D, 3)
    Id = torch.from_numpy(I.astype(np.float32)).to(dev).bfloat16()
    Td = torch.from_numpy(T.astype(np.float32)).to(dev).bfloat16()
    (di0, dt0, l0), ms0 = run(Id, Td, False, a.reps)
    (di1, dt1, l1), ms1 = run(Id, Td, True, a.reps)
    di0, dt0, di1, dt1 = (x.cpu().numpy() for x in (di0, dt0, di1, dt1))
    Ib, Tb = O.bf16_round(I), O.bf16_round(T)
    rows = np.linspace(0, B - 1, 24).astype(np.int64)
    ri, rt, rl = O.clip_grad_rows(Ib, Tb, a.t, rows)
    r = {"ms_off": round(ms0, 4), "ms_on": round(ms1, 4),
         "on_vs_off": [float(O.max_rel_error(di1, di0)), float(O.max_rel_error(dt1, dt0)), abs(l1 - l0) / abs(l0)],
         "on_vs_oracle": [float(O.max_rel_error(di1[rows], ri)), float(O.max_rel_error(dt1[rows], rt)),
                           abs(l1 - rl[0]) / rl[0]],
         "off_vs_oracle": [float(O.max_rel_error(di0[rows], ri)), float(O.max_rel_error(dt0[rows], rt)),
                                abs(l0 - rl[0]) / rl[0]],
         "bitwise_d_image": bool(np.array_equal(di0, di1)), "bitwise_d_text": bool(np.array_equal(dt0, dt1))}
    res[sz] = r
    print(sz, json.dumps(r), flush=True)
    os.environ.pop(a.var, None)
print(json.dumps(res))
