"""Loss-scope memory / FLOP accounting, measured on the B200.

Mirrors the reference cost model (/root/reference/pkg/src/disco/costs.py):

  CostInputs, CostReport, CSV_FIELDS      costs.py:42-94
  analytic_footprint                      costs.py:97-113 (exact per-rank formulas)
  savings_fraction                        costs.py:116-121
  measured_footprint / measured_detail    costs.py:124-187
  bytes_moved                             costs.py:190-197
  reports_to_csv / _json / _table         costs.py:200-223

The analytic side is the same integer arithmetic.  The measured side runs
the real device path instead of the instrumented numpy one: ``disco`` mode
runs this package's sm_100a ``disco_step`` with N simulated ranks on one GPU
and ``naive`` mode a full-batch CLIP loss (one B x B fp32 logit matrix and
its autograd backward, torch on the same GPU).  ``bytes`` is the device
memory the loss call allocated per rank (torch caching-allocator peak over a
clean slate), not an element count times a scalar size; ``loss_elements`` /
``loss_flops`` keep the reference's conventions (2*b*B loss elements for
DisCo, B*B for CLIP; 2 FLOPs per multiply-add in measured reports).

    python -m paper_2304_08480_b200.costs --batch-size 32768 --world-size 8 --dim 512
"""

import argparse
import csv
import io
import json
import sys
from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import torch

from .errors import DomainError
from .fabric import CONCURRENT, LOCKSTEP

METHODS = ("CLIP", "BASIC", "DisCo", "DisCo*")
CSV_FIELDS = ("method", "B", "N", "L", "D", "backbone_elements",
              "loss_elements", "total_elements", "loss_flops", "bytes")
PRECISION_BYTES = {"f32": 4, "f64": 8}


@dataclass(frozen=True)
class CostInputs:
    B: int
    N: int
    L: int
    D: int
    bytes_per_scalar: int

    def __post_init__(self):
        for name in ("B", "N", "L", "D"):
            if getattr(self, name) < 1:
                raise DomainError(f"{name} must be >= 1, got {getattr(self, name)}")
        if self.B % self.N != 0:
            raise DomainError(f"B={self.B} is not divisible by N={self.N}")
        if self.bytes_per_scalar not in (4, 8):
            raise DomainError(f"bytes per scalar must be 4 or 8, got {self.bytes_per_scalar}")


@dataclass(frozen=True)
class CostReport:
    method: str
    B: int
    N: int
    L: int
    D: int
    backbone_elements: int
    loss_elements: int
    total_elements: int
    loss_flops: int
    bytes: int

    def __post_init__(self):
        if self.total_elements != self.backbone_elements + self.loss_elements:
            raise ValueError("total_elements must equal backbone + loss elements")

    def as_row(self) -> dict:
        return {name: getattr(self, name) for name in CSV_FIELDS}


def _report(method, B, N, L, D, backbone, loss_elements, loss_flops, nbytes) -> CostReport:
    return CostReport(method=method, B=B, N=N, L=L, D=D, backbone_elements=backbone,
                      loss_elements=loss_elements, total_elements=backbone + loss_elements,
                      loss_flops=loss_flops, bytes=nbytes)


def analytic_footprint(inputs: CostInputs, method: str) -> CostReport:
    """Per-rank elements and FLOPs (costs.py:97-113): activations of the b local rows
    (all L layers, or one with recomputation for BASIC / DisCo*), one B x B logit
    matrix (CLIP, BASIC) or two b x B blocks (DisCo, DisCo*), 1 FLOP per multiply-add."""
    if method not in METHODS:
        raise DomainError(f"method must be one of {METHODS}, got {method!r}")
    B, N, L, D = inputs.B, inputs.N, inputs.L, inputs.D
    b = B // N
    backbone = b * L * D if method in ("CLIP", "DisCo") else b * D
    if method in ("CLIP", "BASIC"):
        loss_elements, loss_flops = B * B, B * B * D
    else:
        loss_elements, loss_flops = 2 * B * B // N, 2 * B * B * D // N
    total = backbone + loss_elements
    return _report(method, B, N, L, D, backbone, loss_elements, loss_flops, total * inputs.bytes_per_scalar)


def savings_fraction(N: int) -> Fraction:
    """Loss-scope memory saved by sharding, max(0, 1 - 2/N) exactly (costs.py:116-121)."""
    if N < 1:
        raise DomainError(f"N must be >= 1, got {N}")
    return max(Fraction(0), 1 - Fraction(2, N))


def bytes_moved(collective: str, buffer_elements: int, N: int) -> int:
    """Elements received per rank, N blocks for either collective (costs.py:190-197)."""
    if collective not in ("all_gather", "all_reduce"):
        raise DomainError(f"collective must be 'all_gather' or 'all_reduce', got {collective!r}")
    if buffer_elements < 0 or N < 1:
        raise DomainError(f"invalid sizes: buffer_elements={buffer_elements}, N={N}")
    return N * buffer_elements


# ---------------------------------------------------------------------------
# measured on the device
# ---------------------------------------------------------------------------
def _features(B, D, seed, device, dtype=torch.float32):
    """cli.py:103-105 inputs (seeded, rows L2-normalised), on the device."""
    rng = np.random.default_rng(seed)
    I = rng.standard_normal((B, D))
    I /= np.linalg.norm(I, axis=1, keepdims=True)
    T = rng.standard_normal((B, D))
    T /= np.linalg.norm(T, axis=1, keepdims=True)
    return (torch.tensor(I, dtype=dtype, device=device),
            torch.tensor(T, dtype=dtype, device=device))


def _naive_clip_step(I, T, t):
    """Full-batch CLIP loss + feature gradients on one GPU (the replicated baseline)."""
    I = I.detach().requires_grad_(True)
    T = T.detach().requires_grad_(True)
    S = (I @ T.t()) * t
    labels = torch.arange(S.shape[0], device=S.device)
    loss = 0.5 * (torch.nn.functional.cross_entropy(S, labels) + torch.nn.functional.cross_entropy(S.t(), labels))
    loss.backward()
    return I.grad, T.grad, float(loss.detach())




def _validate_measured(mode, B, N, precision, scheduler):
    if mode not in ("naive", "disco"):
        raise DomainError(f"mode must be 'naive' or 'disco', got {mode!r}")
    if precision not in PRECISION_BYTES:
        raise DomainError(f"precision must be one of {tuple(PRECISION_BYTES)}")
    if scheduler not in (LOCKSTEP, CONCURRENT):
        raise DomainError(f"scheduler must be {LOCKSTEP!r} or {CONCURRENT!r}, got {scheduler!r}")
    if B % N != 0:
        raise DomainError(f"B={B} is not divisible by N={N}")
    if not torch.cuda.is_available():
        raise RuntimeError("measured footprints need a CUDA device (no CPU fallback)")


def measured_detail(mode: str, B: int, N: int, D: int, *, precision: str = "f64", temperature: float = 10.0,
                    seed: int = 0, scheduler: str = LOCKSTEP, device=None):
    """Raw per-rank counter peaks (loss_peak, loss_flops, exchange_peak) -- costs.py:143-187.

    Same contract as the reference: ``disco`` passes ``Counters`` through this package's
    ``disco_step`` on N simulated ranks (the device path records the reference's accounting,
    shard.py:133-156 and 192-204: loss peak 2*b*B, 4*b*B*D FLOPs, exchange peak 5*B*D) and
    returns the max over ranks; ``naive`` runs the full-batch CLIP loss on the GPU with the
    accounting of clip_grad_full (oracle.py:148-186: B*B, 2*B*B*D, 2*B*D).  The device bytes
    the call allocates are ``measured_device_bytes``.
    """
    from . import shard
    from .counters import Counters
    from .fabric import run_ranks

    _validate_measured(mode, B, N, precision, scheduler)
    device = device or torch.device("cuda", torch.cuda.current_device())
    I, T = _features(B, D, seed, device, torch.float64 if precision == "f64" else torch.float32)
    if mode == "naive":
        loss_counters, exchange_counters = Counters(), Counters()
        loss_counters.add_flops(2 * B * B * D)
        loss_counters.alloc(B * B)
        _naive_clip_step(I, T, temperature)
        exchange_counters.add_flops(4 * B * B * D)
        exchange_counters.alloc(2 * B * D)
        loss_counters.release(B * B)
        return (loss_counters.peak_live_elements, loss_counters.flops, exchange_counters.peak_live_elements)
    b = B // N

    def fn(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        lc, xc = Counters(), Counters()
        shard.disco_step(ep, I[rows], T[rows], temperature, loss_counters=lc, exchange_counters=xc)
        return lc.peak_live_elements, lc.flops, xc.peak_live_elements

    per_rank = run_ranks(N, fn, device=device)
    return tuple(max(v) for v in zip(*per_rank))


def measured_device_bytes(mode: str, B: int, N: int, D: int, *, temperature: float = 10.0, seed: int = 0,
                          device=None) -> int:
    """Device bytes one loss call allocates per rank (torch caching-allocator peak over a clean slate).

    disco: N simulated ranks (threads) run ``disco_step`` on fresh workspaces; the peak divided by
    N (the ranks are symmetric) is the per-rank footprint, plus the rank's peer window (cudaMalloc'd
    outside torch, N > 1 with the peer transport).  naive: one full-batch CLIP step.
    """
    from . import shard
    from .fabric import run_ranks

    _validate_measured(mode, B, N, "f32", LOCKSTEP)
    device = device or torch.device("cuda", torch.cuda.current_device())
    I, T = _features(B, D, seed, device)
    shard.clear_plans()
    torch.cuda.synchronize(device)
    torch.cuda.empty_cache()
    base = torch.cuda.memory_allocated(device)
    torch.cuda.reset_peak_memory_stats(device)
    if mode == "naive":
        _naive_clip_step(I, T, temperature)
        torch.cuda.synchronize(device)
        per_rank = torch.cuda.max_memory_allocated(device) - base
    else:
        b = B // N

        def fn(ep):
            rows = slice(ep.rank * b, (ep.rank + 1) * b)
            return shard.disco_step(ep, I[rows], T[rows], temperature)[2]

        run_ranks(N, fn, device=device)
        torch.cuda.synchronize(device)
        per_rank = (torch.cuda.max_memory_allocated(device) - base) // N
        per_rank += peer_window_bytes(B, D, N)
    shard.clear_plans()
    torch.cuda.empty_cache()
    return int(per_rank)


def peer_window_bytes(B: int, D: int, N: int, rank: int = 0) -> int:
    """Bytes of a rank's peer-transport window (0 when the geometry does not use it)."""
    import ctypes
    from . import _lib
    from . import peer

    if not peer.supported(B, D, N, rank):
        return 0
    out = ctypes.c_int64()
    _lib.call("disco_b200_peer_bytes", B, D, N, rank, ctypes.byref(out))
    return int(out.value)


def measured_footprint(mode: str, B: int, N: int, D: int, *, precision: str = "f64", temperature: float = 10.0,
                       seed: int = 0, scheduler: str = LOCKSTEP, device=None) -> CostReport:
    """CostReport of one measured loss call (costs.py:124-140 schema).  ``loss_elements`` /
    ``loss_flops`` are the counter peaks of ``measured_detail``; ``bytes`` is the MEASURED device
    footprint per rank (``measured_device_bytes``), not elements x scalar size."""
    le, lf, _ = measured_detail(mode, B, N, D, precision=precision, temperature=temperature, seed=seed,
                                scheduler=scheduler, device=device)
    nbytes = measured_device_bytes(mode, B, N, D, temperature=temperature, seed=seed, device=device)
    return _report("CLIP" if mode == "naive" else "DisCo", B, N, 0, D, 0, le, lf, nbytes)


def reports_to_csv(reports) -> str:
    out = io.StringIO()
    w = csv.DictWriter(out, fieldnames=CSV_FIELDS, lineterminator="\n")
    w.writeheader()
    for r in reports:
        w.writerow(r.as_row())
    return out.getvalue()


def reports_to_json(reports) -> str:
    return json.dumps([r.as_row() for r in reports], indent=2) + "\n"


def reports_to_table(reports) -> str:
    rows = [[str(v) for v in r.as_row().values()] for r in reports]
    widths = [max([len(CSV_FIELDS[i])] + [len(row[i]) for row in rows]) for i in range(len(CSV_FIELDS))]
    lines = ["  ".join(n.ljust(widths[i]) for i, n in enumerate(CSV_FIELDS))]
    lines += ["  ".join(c.ljust(widths[i]) for i, c in enumerate(row)) for row in rows]
    return "\n".join(lines) + "\n"


def main(argv=None) -> int:
    """`disco bench` on the GPU (cli.py:203-224): measured per-rank footprints."""
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--batch-size", type=int, default=4096)
    ap.add_argument("--world-size", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--dim", type=int, default=512)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--mode", choices=("naive", "disco", "both"), default="both")
    ap.add_argument("--format", choices=("csv", "json", "table"), default="table")
    a = ap.parse_args(argv)
    modes = ["naive", "disco"] if a.mode == "both" else [a.mode]
    reports = []
    for mode in modes:
        for N in (a.world_size if mode == "disco" else [1]):
            reports.append(measured_footprint(mode, a.batch_size, N, a.dim, seed=a.seed))
    fmt = {"csv": reports_to_csv, "json": reports_to_json, "table": reports_to_table}[a.format]
    sys.stdout.write(fmt(reports))
    return 0


if __name__ == "__main__":
    sys.exit(main())
