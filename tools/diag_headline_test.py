"""pytest-context replica of test_headline_shape_bitwise_across_world_sizes with per-rank failure
details (flags, time, gathered-operand mismatches by source rank).  Run explicitly:
  python -m pytest tools/diag_headline_test.py -s -q -p no:cacheprovider"""
import os
import sys
import time

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import paper_2304_08480_b200 as P  # noqa: E402
from paper_2304_08480_b200 import _lib  # noqa: E402
from paper_2304_08480_b200.shard import clear_plans, get_plan, _read_status  # noqa: E402
from oracle import disco_oracle as O  # noqa: E402


@pytest.mark.parametrize("rep", range(3))
@pytest.mark.parametrize("peer", [False, True], ids=["nccl", "peer"])
def test_replica(peer, rep):
    clear_plans()
    torch.cuda.empty_cache()
    B, D, t = 32768, 512, 100.0
    I, T = O.synthetic_features(B, D, 7)
    Id = torch.from_numpy(np.ascontiguousarray(I, dtype=np.float32)).cuda()
    Td = torch.from_numpy(np.ascontiguousarray(T, dtype=np.float32)).cuda()
    ref = torch.stack([Id.bfloat16(), Td.bfloat16()])
    di1, dt1, l1 = P.disco_step(None, Id, Td, t)
    bad_any = []
    for N in (2, 4, 8):
        clear_plans()
        b = B // N

        def fn(ep):
            t0 = time.time()
            rows = slice(ep.rank * b, (ep.rank + 1) * b)
            try:
                P.disco_step(ep, Id[rows], Td[rows], t)
                return None
            except Exception as exc:
                torch.cuda.current_stream().synchronize()
                el = time.time() - t0
                plan = get_plan(B, D, N, ep.rank, Id.device)
                _, flags = _read_status(plan)
                feat = plan.feat[:, :, :D]
                per_src = (feat != ref).any(2).view(2, N, b).sum(2).cpu().tolist()
                off, size = _lib.ws_region(B, D, N, ep.rank, _lib.R_FEAT16)
                f16 = plan.ws[off:off + size].view(torch.float16).view(2, B, plan.Dp)[:, :, :D]
                nf16 = int((~torch.isfinite(f16)).sum())
                off, size = _lib.ws_region(B, D, N, ep.rank, _lib.R_INTRA)
                nint = int((~torch.isfinite(plan.ws[off:off + size].view(torch.float32))).sum())
                off, size = _lib.ws_region(B, D, N, ep.rank, _lib.R_G)
                nE = int((~torch.isfinite(plan.ws[off:off + size].view(torch.float16))).sum())
                return dict(rank=ep.rank, exc=repr(exc)[:80], flags=flags, sec=round(el, 2), feat_bad=per_src,
                            f16_nonfinite=nf16, intra_nonfinite=nint, E_nonfinite=nE, fixed=plan.fixed_rows)

        t0 = time.time()
        res = P.run_ranks(N, fn, peer=peer)
        fails = [x for x in res if x is not None]
        print(f"\n{'peer' if peer else 'nccl'} rep={rep} N={N} {time.time() - t0:.2f}s fails={fails}", flush=True)
        bad_any += fails
    assert not bad_any
