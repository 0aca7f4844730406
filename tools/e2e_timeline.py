"""GPU timeline of the end-to-end (host buffers) disco_step: kernels and copies per stream.

  python tools/e2e_timeline.py [--batch 32768] [--dim 512] [--out gpurun_out/e2e_trace.json]

Runs the public disco_step with pinned bf16 host features (bench.py's e2e leg) under
torch.profiler (CUPTI activity records; a profiling aid, never a bench value) and prints,
for the last step, every GPU activity with its start / end relative to the first one,
grouped by stream, plus the exposed (non-overlapped) copy time.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32768)
ap.add_argument("--dim", type=int, default=512)
ap.add_argument("--out", default="gpurun_out/e2e_trace.json")
ap.add_argument("--sweep", action="store_true", help="time row-block schedules (CUDA events), no trace")
ap.add_argument("--device", action="store_true", help="device-resident inputs (bench value path) instead of host")
a = ap.parse_args()

torch.cuda.set_device(0)
g = torch.Generator(device="cuda")
g.manual_seed(0)
I = torch.nn.functional.normalize(torch.randn(a.batch, a.dim, device="cuda", generator=g), dim=1)
T = torch.nn.functional.normalize(torch.randn(a.batch, a.dim, device="cuda", generator=g), dim=1)
I_h = I.bfloat16() if a.device else I.bfloat16().cpu().pin_memory()
T_h = T.bfloat16() if a.device else T.bfloat16().cpu().pin_memory()
for _ in range(3):
    P.disco_step(None, I_h, T_h, 100.0)
torch.cuda.synchronize()
if a.sweep:
    import statistics
    from paper_2304_08480_b200 import shard
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    schedules = [shard.ROW_BLOCK_FRACTIONS, (0.25, 0.25, 0.25, 0.125, 0.125),
                 (0.0625, 0.1875, 0.25, 0.25, 0.125, 0.0625, 0.0625), (0.125, 0.25, 0.25, 0.25, 0.125),
                 (0.125, 0.1875, 0.1875, 0.1875, 0.1875, 0.125), (0.0625, 0.125, 0.25, 0.25, 0.1875, 0.125)]
    res = {sc: [] for sc in schedules}
    for rep in range(8):
        for sc in schedules:
            shard.ROW_BLOCK_FRACTIONS = sc
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            P.disco_step(None, I_h, T_h, 100.0)
            e1.record()
            e1.synchronize()
            if rep >= 2:
                res[sc].append(e0.elapsed_time(e1))
    for sc, v in res.items():
        print(f"{statistics.median(v):.3f} ms  {sc}")
    sys.exit(0)
marker = torch.empty(1, device="cuda")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for i in range(2):
        marker.fill_(i)  # step boundary in the trace
        P.disco_step(None, I_h, T_h, 100.0)
    torch.cuda.synchronize()
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
prof.export_chrome_trace(a.out)
with open(a.out) as f:
    ev = json.load(f)["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
# the last step: everything after the last marker fill
cut = max(i for i, e in enumerate(gpu) if "fill" in e["name"].lower() or e["cat"] == "gpu_memset")
step = gpu[cut + 1:]
t0 = step[0]["ts"]
end = max(e["ts"] + e["dur"] for e in step)
print(f"step span {(end - t0) / 1e3:.3f} ms, {len(step)} GPU activities")
for e in step:
    s = e["args"].get("stream", "?")
    name = e["name"][:70]
    extra = ""
    if e["cat"] == "gpu_memcpy":
        nb = e["args"].get("bytes", 0)
        extra = f"  {nb / 1e6:.1f} MB @ {nb / e['dur'] / 1e3:.1f} GB/s" if e["dur"] else ""
    print(f"  s{s:>3} {(e['ts'] - t0) / 1e3:8.3f} .. {(e['ts'] + e['dur'] - t0) / 1e3:8.3f} ms  {name}{extra}")
