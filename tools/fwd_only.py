"""Run pack + forward of B=32K, D=512 a few times per given library build (for ncu metric
comparisons of forward variants; never a bench value).  python tools/fwd_only.py a.so b.so ..."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_08480_b200 import _lib  # noqa: E402
from paper_2304_08480_b200.shard import get_plan  # noqa: E402

B, D, t = int(os.environ.get("B", 32768)), int(os.environ.get("D", 512)), 100.0
reps = int(os.environ.get("REPS", 2))
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
    for rep in range(reps):
        flush.zero_()
        lib.disco_b200_pack(*plan.args, I.data_ptr(), T.data_ptr(), D, D, _lib.BF16, 1, sp)
        lib.disco_b200_forward(*plan.args, ctypes.c_float(t), sp)
    torch.cuda.synchronize()
    print(path, "done", flush=True)
