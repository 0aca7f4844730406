"""Print the parity errors of the device path against the f64 oracle for a few shapes.

  python tools/precision_probe.py            (DISCO_RECOMPUTE=1 for the recompute path)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402
from oracle import disco_oracle as O  # noqa: E402

torch.cuda.set_device(0)
for B, D, t, corr in [(1024, 512, 100.0, False), (1024, 512, 100.0, True), (4096, 512, 14.2857, False),
                      (4096, 768, 100.0, True), (8192, 1024, 100.0, False)]:
    I, T = O.synthetic_features(B, D, 0)
    if corr:
        rng = np.random.default_rng(1)
        T = I + 3.0 * rng.standard_normal(I.shape) / np.sqrt(D)
        T /= np.linalg.norm(T, axis=1, keepdims=True)
    Ib, Tb = O.bf16_round(I), O.bf16_round(T)
    di, dt, loss = P.disco_step(None, torch.from_numpy(Ib.astype(np.float32)).cuda(),
                                torch.from_numpy(Tb.astype(np.float32)).cuda(), t)
    ri, rt, rl = O.clip_grad_full(Ib.astype(np.float64), Tb.astype(np.float64), t)
    print(f"B={B} D={D} t={t} corr={corr}: d_image {O.max_rel_error(di.cpu().numpy(), ri):.3e} "
          f"d_text {O.max_rel_error(dt.cpu().numpy(), rt):.3e} loss {abs(loss - rl[0]) / abs(rl[0]):.3e}",
          flush=True)
