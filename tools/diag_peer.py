"""Diagnose the simulated-rank peer path at a given shape: per N, run the step R times with the
peer all-gather and with the endpoint all-gather, report status flags, fixed rows, non-finite
rows and the first differing row versus N = 1.  Never part of a bench value."""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402
from paper_2304_08480_b200.shard import clear_plans  # noqa: E402
from oracle import disco_oracle as O  # noqa: E402


def run(Id, Td, N, t, peer):
    b = Id.shape[0] // N
    info = {}

    def fn(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        try:
            di, dt, loss = P.disco_step(ep, Id[rows], Td[rows], t)
            return di, dt, loss, None
        except Exception as exc:  # keep going: report per rank
            return None, None, None, repr(exc)

    res = P.run_ranks(N, fn, peer=peer)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, default=32768)
    ap.add_argument("--D", type=int, default=512)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--worlds", default="2,4,8")
    a = ap.parse_args()
    t = 100.0
    I, T = O.synthetic_features(a.B, a.D, 7)
    Id = torch.from_numpy(I.astype(np.float32)).cuda()
    Td = torch.from_numpy(T.astype(np.float32)).cuda()
    di1, dt1, l1 = P.disco_step(None, Id, Td, t)
    di1, dt1 = di1.cpu().numpy(), dt1.cpu().numpy()
    print(f"N=1 loss={l1!r} nonfinite={int((~np.isfinite(di1)).sum())}", flush=True)
    for N in [int(x) for x in a.worlds.split(",")]:
        for peer in (True, False):
            for rep in range(a.reps):
                clear_plans()
                res = run(Id, Td, N, t, peer)
                errs = [r[3] for r in res]
                if any(errs):
                    print(f"N={N} peer={peer} rep={rep}: errors {errs}", flush=True)
                    continue
                di = torch.cat([r[0] for r in res]).cpu().numpy()
                dt = torch.cat([r[1] for r in res]).cpu().numpy()
                same_i = di.tobytes() == di1.tobytes()
                same_t = dt.tobytes() == dt1.tobytes()
                bad = np.nonzero((di != di1).any(1) | (dt != dt1).any(1))[0]
                print(f"N={N} peer={peer} rep={rep}: losses={set(r[2] for r in res)} same_i={same_i} "
                      f"same_t={same_t} diff_rows={len(bad)} first={bad[:8].tolist()}", flush=True)


if __name__ == "__main__" and not os.environ.get("DIAG_STRESS"):
    main()


def stress(reps=6, B=32768, D=512):
    """Repeat the peer-mode N = 2, 4, 8 steps; on a failing rank, check its gathered operands."""
    from paper_2304_08480_b200 import _lib
    from paper_2304_08480_b200.shard import get_plan
    t = 100.0
    I, T = O.synthetic_features(B, D, 7)
    Id = torch.from_numpy(I.astype(np.float32)).cuda()
    Td = torch.from_numpy(T.astype(np.float32)).cuda()
    ref = torch.stack([Id.bfloat16(), Td.bfloat16()])  # [2][B][D]
    import time
    for rep in range(reps):
        clear_plans()
        torch.cuda.empty_cache()
        if os.environ.get("DIAG_N1"):
            P.disco_step(None, Id, Td, t)
        if os.environ.get("DIAG_NCCL"):
            for N in (2, 4, 8):
                clear_plans()
                bb = B // N
                P.run_ranks(N, lambda ep: P.disco_step(ep, Id[ep.rank * bb:(ep.rank + 1) * bb],
                                                       Td[ep.rank * bb:(ep.rank + 1) * bb], t))
        for N in (2, 4, 8):
            t0 = time.time()
            clear_plans()
            b = B // N

            def fn(ep):
                rows = slice(ep.rank * b, (ep.rank + 1) * b)
                try:
                    P.disco_step(ep, Id[rows], Td[rows], t)
                    return None
                except Exception as exc:
                    torch.cuda.current_stream().synchronize()
                    plan = get_plan(B, D, N, ep.rank, Id.device)
                    feat = plan.feat[:, :, :D]
                    bad = (feat != ref).any(2)  # [2][B]
                    per_src = bad.view(2, N, b).sum(2).cpu().tolist()
                    off, size = _lib.ws_region(B, D, N, ep.rank, _lib.R_FEAT16)
                    f16 = plan.ws[off:off + size].view(torch.float16).view(2, B, plan.Dp)[:, :, :D]
                    bad16 = (f16.float() != ref.float()).any(2).view(2, N, b).sum(2).cpu().tolist()
                    off, size = _lib.ws_region(B, D, N, ep.rank, _lib.R_INTRA)
                    intra = plan.ws[off:off + size].view(torch.float32)
                    return (repr(exc), per_src, bad16, int((~torch.isfinite(intra)).sum()))

            res = P.run_ranks(N, fn, peer=True)
            fails = [(r, x) for r, x in enumerate(res) if x is not None]
            print(f"stress rep={rep} N={N} {time.time() - t0:.2f}s: {'ok' if not fails else fails}", flush=True)


if __name__ == "__main__" and os.environ.get("DIAG_STRESS"):
    stress(int(os.environ["DIAG_STRESS"]))
