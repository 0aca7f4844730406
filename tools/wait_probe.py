"""Barrier-wait breakdown of the forward logits kernel (profiling build, -DDISCO_WAITPROBE=1):
MMA thread cycles waiting for operand stages (full) and for a free accumulator (tempty), and the
epilogue warps' wait for a finished accumulator (tfull), as fractions of the MMA thread's time.

  python -m paper_2304_08480_b200.build --out abtmp/probe.so -D DISCO_WAITPROBE=1
  python tools/wait_probe.py abtmp/probe.so [more.so ...]
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_08480_b200 import _lib  # noqa: E402
from paper_2304_08480_b200.shard import get_plan  # noqa: E402

B, D, t = int(os.environ.get("B", 32768)), int(os.environ.get("D", 512)), 100.0
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
I = torch.nn.functional.normalize(torch.randn(B, D, device=dev, generator=g), dim=1).bfloat16()
T = torch.nn.functional.normalize(torch.randn(B, D, device=dev, generator=g), dim=1).bfloat16()
plan = get_plan(B, D, 1, 0, dev)
sp = torch.cuda.current_stream(dev).cuda_stream
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for path in sys.argv[1:]:
    lib = ctypes.CDLL(os.path.abspath(path))
    for name, argtypes in _lib.SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is not None:
            fn.argtypes = argtypes
            fn.restype = _lib._RESTYPES.get(name, ctypes.c_int)
    out = (ctypes.c_ulonglong * 16)()
    for rep in range(25):
        if rep == 5:
            torch.cuda.synchronize()
            lib.disco_b200_waitprobe(out, 1)
        flush.zero_()
        lib.disco_b200_pack(*plan.args, I.data_ptr(), T.data_ptr(), D, D, _lib.BF16, 1, sp)
        lib.disco_b200_forward(*plan.args, ctypes.c_float(t), sp)
        lib.disco_b200_dual_prep(*plan.args, 0, sp)
        lib.disco_b200_backward_dual(*plan.args, 0, B, sp)
    torch.cuda.synchronize()
    lib.disco_b200_waitprobe(out, 0)
    v = list(out)
    tot = v[2] or 1
    print(f"{os.path.basename(path)}: MMA threads {v[3]}  full-wait {v[0] / tot:.3f}  tempty-wait {v[1] / tot:.3f}  "
          f"epilogue tfull-wait {[round(x / (tot * 4), 3) for x in v[4:8]]} (per quadrant, / MMA time)")
    gt, xt = v[10] or 1, v[13] or 1
    print(f"   backward GEMM: MMA threads {v[11]}  operand (xfull) wait {v[8] / gt:.3f}  tempty wait {v[9] / gt:.3f};  "
          f"transform warps {v[14]}  TMA (full) wait {v[12] / xt:.3f}")
