"""Host-side cost of one disco_step_async enqueue (no device sync) vs its device time, at N = 1
on device-resident bf16 features; the enqueue rate bounds small per-rank steps (N = 8).
  python tools/host_overhead.py [B ...]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402

dev = torch.device("cuda", 0)
for B in [int(x) for x in sys.argv[1:]] or [4096, 32768]:
    D = 512
    I = torch.nn.functional.normalize(torch.randn(B, D, device=dev), dim=1).bfloat16()
    T = torch.nn.functional.normalize(torch.randn(B, D, device=dev), dim=1).bfloat16()
    ep = P.SingleEndpoint()
    for _ in range(5):
        P.disco_step_async(ep, I, T, 100.0)
    torch.cuda.synchronize()
    n = 50
    # host cost with the GPU far behind (queue filling): time to enqueue n steps
    t0 = time.perf_counter()
    for _ in range(n):
        P.disco_step_async(ep, I, T, 100.0)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        P.disco_step_async(ep, I, T, 100.0)
    e1.record()
    torch.cuda.synchronize()
    print(f"B={B}: host enqueue {(t1 - t0) / n * 1e3:.3f} ms/step, wall {(t2 - t0) / n * 1e3:.3f} ms/step, "
          f"device back-to-back {e0.elapsed_time(e1) / n:.3f} ms/step", flush=True)
    P.clear_plans() if hasattr(P, "clear_plans") else None
