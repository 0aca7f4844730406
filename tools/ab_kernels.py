"""Same-process A/B timing of kernel variants (profiling experiments, not a bench value).

Alternates experiment-flag settings (disco_b200_set_experiment_flags) rep by rep so every
variant sees the same clocks / thermal state, and reports the median per-phase time.

  python tools/ab_kernels.py --flags 0 128 --reps 15
  python tools/ab_kernels.py --so-b /path/to/other/_disco_b200.so   (two builds, same ABI)
"""
import argparse
import ctypes
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402
from paper_2304_08480_b200 import _lib  # noqa: E402
from paper_2304_08480_b200.shard import get_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32768)
ap.add_argument("--dim", type=int, default=512)
ap.add_argument("--flags", type=int, nargs="+", default=[0])
ap.add_argument("--so-b", default=None, help="second library build to alternate with")
ap.add_argument("--so", nargs="*", default=[], help="more library builds to alternate with (name=path or path)")
ap.add_argument("--reps", type=int, default=15)
ap.add_argument("--warm", type=float, default=3.0, help="seconds of untimed steps first (clocks ramp)")
ap.add_argument("--exchange", action="store_true", help="time the exchange backward instead of the dual one")
a = ap.parse_args()

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
B, D, t = a.batch, a.dim, 100.0
g = torch.Generator(device=dev)
g.manual_seed(0)
I = torch.nn.functional.normalize(torch.randn(B, D, device=dev, generator=g), dim=1).bfloat16()
T = torch.nn.functional.normalize(torch.randn(B, D, device=dev, generator=g), dim=1).bfloat16()
plan = get_plan(B, D, 1, 0, dev)
# experiments may change the geometry (e.g. bit8 narrow units): give the workspace the max size
_need = 0
for _f in a.flags:
    _lib.load().disco_b200_set_experiment_flags(_f)
    _need = max(_need, _lib.workspace_bytes(B, D, 1, 0))
_lib.load().disco_b200_set_experiment_flags(0)
if _need > plan.ws.numel():
    plan.ws = torch.empty(_need, dtype=torch.uint8, device=dev)
    plan.ptr = plan.ws.data_ptr()
st = torch.cuda.current_stream(dev)
sp = st.cuda_stream
di = torch.empty((B, D), dtype=torch.float32, device=dev)
dt = torch.empty((B, D), dtype=torch.float32, device=dev)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

libs = [("main", _lib.load())]
extra = ([("b", a.so_b)] if a.so_b else []) + [
    (x.split("=", 1)[0], x.split("=", 1)[1]) if "=" in x else (os.path.basename(x).rsplit(".", 1)[0], x) for x in a.so]
for lname, path in extra:
    lb = ctypes.CDLL(os.path.abspath(path))
    for name, argtypes in _lib.SIGNATURES.items():
        fn = getattr(lb, name, None)
        if fn is None:  # older build: no experiment-flag hook
            continue
        fn.argtypes = argtypes
        fn.restype = _lib._RESTYPES.get(name, ctypes.c_int)
    libs.append((lname, lb))
variants = [(ln, lib, f) for ln, lib in libs for f in a.flags]


def run(lib, flags, ev):
    if hasattr(lib, "disco_b200_set_experiment_flags"):
        lib.disco_b200_set_experiment_flags(flags)
    args = plan.args
    assert lib.disco_b200_pack(*args, I.data_ptr(), T.data_ptr(), D, D, _lib.BF16, 1, sp) == 0
    ev[0].record(st)
    assert lib.disco_b200_forward(*args, t, sp) == 0
    ev[1].record(st)
    if a.exchange:
        assert lib.disco_b200_backward_grad(*args, t, sp) == 0
        assert lib.disco_b200_backward_fused(*args, sp) == 0
        ev[2].record(st)
        assert lib.disco_b200_combine(*args, t, 0, di.data_ptr(), dt.data_ptr(), D, sp) == 0
    else:
        assert lib.disco_b200_dual_prep(*args, 0, sp) == 0
        assert lib.disco_b200_backward_dual(*args, 0, B, sp) == 0
        ev[2].record(st)
        assert lib.disco_b200_combine_dual(*args, t, 0, B, di.data_ptr(), dt.data_ptr(), D, sp) == 0
    ev[3].record(st)


import time as _time
_t0 = _time.time()
while _time.time() - _t0 < a.warm:
    run(libs[0][1], a.flags[0], [torch.cuda.Event(enable_timing=True) for _ in range(4)])
    torch.cuda.synchronize()
times = {v[0] + ":" + str(v[2]): ([], [], []) for v in variants}
mhz = {}
for rep in range(a.reps + 2):
    for ln, lib, f in variants:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        flush.zero_()
        run(lib, f, ev)
        torch.cuda.synchronize()
        if rep >= 2:
            k = ln + ":" + str(f)
            for i in range(3):
                times[k][i].append(ev[i].elapsed_time(ev[i + 1]))
            mhz.setdefault(k, []).append(_lib.clock_probe(plan))
for k, (fw, bw, cb) in times.items():
    mf = statistics.median(m['logits_fwd'] for m in mhz[k])
    mb = statistics.median(m['gemm_backward'] for m in mhz[k])
    print(f"{k:10s} cycles(k) fwd {statistics.median(fw) * mf:.0f} bwd {statistics.median(bw) * mb:.0f}   "
          f"forward {statistics.median(fw):.4f}  backward {statistics.median(bw):.4f}  "
          f"combine {statistics.median(cb):.4f}  total {statistics.median(fw) + statistics.median(bw) + statistics.median(cb):.4f} ms"
          f"  SM MHz fwd {statistics.median(m['logits_fwd'] for m in mhz[k]):.0f} "
          f"bwd {statistics.median(m['gemm_backward'] for m in mhz[k]):.0f} "
          f"drain {statistics.median(m['drain_cycles_per_unit'] for m in mhz[k]):.0f} cyc/unit")
