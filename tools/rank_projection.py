"""Per-rank device time of one DisCo step at world size N, measured on ONE GPU (a projection aid).

  python tools/rank_projection.py [--batch 32768] [--dim 512] [--worlds 1 2 4 8] [--reps 10]

For each N this runs rank 0's share of the default (dual-backward) step on the local GPU --
pack, unpack of a gathered buffer (filled once, untimed: the all_gather itself is NOT measured),
the forward, the statistics "all_gather" (rank 0's 4 b statistics copied into every slot), the
column factors, the dual backward GEMM, the combine, the fixup and the loss -- and reports the
per-phase CUDA-event times, the per-rank FLOP rate (the reference's 12 b B D) and the
compute-only projection B / t_rank.  The collectives are absent, so this is an upper bound on
multi-GPU throughput, not a multi-GPU measurement.
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402,F401
from paper_2304_08480_b200 import _lib  # noqa: E402
from paper_2304_08480_b200.shard import clear_plans, get_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32768)
ap.add_argument("--dim", type=int, default=512)
ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--t", type=float, default=100.0)
ap.add_argument("--flags", type=int, nargs="+", default=[0], help="experiment flag settings to compare per N")
a = ap.parse_args()
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
B, D, t = a.batch, a.dim, a.t
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream(dev)
sp = st.cuda_stream
out = {}
for N, flags in [(N, f) for N in a.worlds for f in a.flags]:
    _lib.load().disco_b200_set_experiment_flags(flags)
    clear_plans()
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats(dev)
    mem0 = torch.cuda.memory_allocated(dev)
    b = B // N
    plan = get_plan(B, D, N, 0, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(N)
    I = torch.nn.functional.normalize(torch.randn(b, D, device=dev, generator=g), dim=1).bfloat16()
    T = torch.nn.functional.normalize(torch.randn(b, D, device=dev, generator=g), dim=1).bfloat16()
    args = plan.args
    di = torch.empty((b, D), dtype=torch.float32, device=dev)
    dt = torch.empty((b, D), dtype=torch.float32, device=dev)
    if N > 1:
        # the gathered buffer: every rank's packed rows (random unit vectors), filled once
        plan.gather.copy_(torch.nn.functional.normalize(
            torch.randn(N * 2 * b, plan.Dp, device=dev, generator=g), dim=1).bfloat16().view(-1))
    phases = ["pack", "forward", "stats", "backward", "combine", "loss"]
    acc = {k: [] for k in phases + ["step"]}
    for rep in range(a.reps + 3):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(phases) + 1)]
        ev[0].record(st)
        _lib.call("disco_b200_pack", *args, I.data_ptr(), T.data_ptr(), D, D, _lib.BF16, 1, sp)
        ev[1].record(st)
        _lib.call("disco_b200_forward", *args, t, sp)
        ev[2].record(st)
        if N > 1:  # stand-in for the 16 b-byte statistics all_gather: rank 0's vector in every slot
            plan.xall.view(N, -1).copy_(plan.xchg.view(1, -1).expand(N, -1))
        _lib.call("disco_b200_dual_prep", *args, 0, sp)
        ev[3].record(st)
        _lib.call("disco_b200_backward_dual", *args, 0, b, sp)
        ev[4].record(st)
        _lib.call("disco_b200_combine_dual", *args, t, 0, b, di.data_ptr(), dt.data_ptr(), D, sp)
        _lib.call("disco_b200_dual_fixup", *args, t, 0, di.data_ptr(), dt.data_ptr(), D, sp)
        ev[5].record(st)
        _lib.call("disco_b200_loss", *args, 2, sp)
        ev[6].record(st)
        torch.cuda.synchronize()
        if rep >= 3:
            for k, name in enumerate(phases):
                acc[name].append(ev[k].elapsed_time(ev[k + 1]))
            acc["step"].append(ev[0].elapsed_time(ev[-1]))
    med = {k: round(statistics.median(v), 4) for k, v in acc.items()}
    flops = 12.0 * b * B * D
    mhz = _lib.clock_probe(plan)
    out[f"{N}:{flags}"] = {"peak_rank_mem_gb": round((torch.cuda.max_memory_allocated(dev) - mem0) / 1e9, 2), "ms": med, "rank_tflops": round(flops / (med["step"] / 1e3) / 1e12, 1),
              "projected_samples_per_s": round(B / (med["step"] / 1e3)), "in_kernel_mhz": mhz}
    o = out[f"{N}:{flags}"]
    print(f"N={N} flags={flags}: step {med['step']:.3f} ms/rank  {o['rank_tflops']} TF/s/rank  "
          f"compute-only projection {o['projected_samples_per_s'] / 1e6:.2f} M samples/s  {med}  MHz {mhz}", flush=True)
print(json.dumps({"batch": B, "dim": D, "note": "rank 0 of N on one GPU; collectives not measured", "worlds": out}))
