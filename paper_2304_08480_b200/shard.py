"""Per-rank DisCo loss on B200: the drop-in for reference shard.py.

Same names, arguments, validation order and exceptions as the reference
(/root/reference/pkg/src/disco/shard.py):

  ShardLayout            shard.py:30-58
  LocalGradContribution  shard.py:61-80
  shard_slice            shard.py:83-89
  local_labels           shard.py:92-95
  local_loss_and_grads   shard.py:98-166
  disco_step             shard.py:169-208

The arithmetic runs in the sm_100a kernels behind the C ABI
(include/disco_b200.h); this module only validates, allocates the
workspace, sequences the stream-ordered calls and issues the collectives
through the endpoint.  There is no CPU fallback.

Dataflow of ``disco_step`` on rank n (b = B/N):
  pack (bf16)  -> all_gather [N][2][b][Dp]   (shard.py:190-191)
  forward      : fused logits GEMM + online LSE + CE, stores E = exp2(y - group max) in f16
                 (shard.py:134-141); host inputs at N = 1: chunked H2D + logit wavefronts
  backward_grad : no-op for canonical shapes (G = softmax - onehot is formed from E inside the
                 backward GEMMs' shared-memory stages); otherwise recompute (shard.py:143-146)
  backward     : intra G . gathered feats and cross G^T . local feats per canonical chunk in one
                 persistent launch (shard.py:149-152); at N > 1 the cross tiles are pushed into
                 the owners' peer windows by the GEMM epilogue (peer transport), or presummed
                 and exchanged with an NCCL all_to_all (DISCO_PEER=0)      \\  replace
  combine      : s * (intra + fixed-tree sum of the chunk partials)         /  all_reduce(AVG)
                 (host outputs at N = 1: row blocks with overlapped D2H)       + row slice
  all_gather of per-row ce -> fixed-order f64 loss (shard.py:205)              (shard.py:199-208)
"""

from dataclasses import dataclass
import os
import threading

import numpy as np
import torch

from . import _lib
from . import peer as _peer
from .counters import Counters, tracking
from .errors import CollectiveTimeoutError, DomainError, LayoutError, ShapeError
from .fabric import SingleEndpoint


@dataclass(frozen=True)
class ShardLayout:
    """Which contiguous slice of the global batch a rank owns (shard.py:30-58)."""

    world_size: int
    global_batch: int
    rank: int

    def __post_init__(self):
        if self.world_size < 1:
            raise LayoutError(f"world size must be >= 1, got {self.world_size}")
        if self.global_batch < 1:
            raise LayoutError(f"global batch must be >= 1, got {self.global_batch}")
        if self.global_batch % self.world_size != 0:
            raise LayoutError(
                f"global batch {self.global_batch} is not divisible by "
                f"world size {self.world_size}")
        if not 0 <= self.rank < self.world_size:
            raise LayoutError(f"rank {self.rank} outside [0, {self.world_size})")

    @property
    def local_batch(self) -> int:
        return self.global_batch // self.world_size

    @property
    def row_slice(self) -> slice:
        start = self.rank * self.local_batch
        return slice(start, start + self.local_batch)


@dataclass(frozen=True)
class LocalGradContribution:
    """One rank's full-size (B x D, fp32) additive contribution (shard.py:61-80).

    Finiteness is checked on the device (status flags) before construction.
    """

    d_image_full: object
    d_text_full: object
    local_loss: float

    def __post_init__(self):
        if tuple(self.d_image_full.shape) != tuple(self.d_text_full.shape):
            raise ShapeError(
                f"contribution shapes disagree: {tuple(self.d_image_full.shape)} "
                f"vs {tuple(self.d_text_full.shape)}")


def shard_slice(layout: ShardLayout, full):
    """Rows [n*b, (n+1)*b) of a global matrix, as a view (shard.py:83-89)."""
    if full.shape[0] != layout.global_batch:
        raise LayoutError(
            f"matrix has {full.shape[0]} rows, layout expects {layout.global_batch}")
    return full[layout.row_slice]


def local_labels(layout: ShardLayout) -> np.ndarray:
    """Global column indices of the rank's positive pairs: arange(b) + b*rank (shard.py:92-95)."""
    b = layout.local_batch
    return np.arange(b) + b * layout.rank


# ---------------------------------------------------------------------------
# Workspace plan
# ---------------------------------------------------------------------------
_TORCH_DTYPE_CODE = {
    torch.float32: _lib.F32,
    torch.bfloat16: _lib.BF16,
    torch.float64: _lib.F64,
    torch.float16: _lib.F16,
}


class Plan:
    """Device workspace + typed views for one (B, D, N, rank, device) geometry."""

    def __init__(self, B: int, D: int, world: int, rank: int, device: torch.device):
        self.B, self.D, self.world, self.rank, self.device = B, D, world, rank, device
        self.b = B // world
        self.Dp = (D + 63) // 64 * 64
        self.nchunk, self.cpr = _lib.chunking(B, world)
        nbytes = _lib.workspace_bytes(B, D, world, rank)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
        self.ptr = self.ws.data_ptr()

        def view(region, dtype):
            off, size = _lib.ws_region(B, D, world, rank, region)
            return self.ws[off:off + size].view(dtype)

        self.pack = view(_lib.R_PACK, torch.bfloat16)
        self.gather = view(_lib.R_GATHER, torch.bfloat16)
        self.ce = view(_lib.R_CE, torch.float32)
        self.ce_all = view(_lib.R_CE_ALL, torch.float32)
        self.send = view(_lib.R_SEND, torch.float32)
        self.recv = view(_lib.R_RECV, torch.float32)
        self.rdot = view(_lib.R_RDOT, torch.float32)
        self.rdot_all = view(_lib.R_RDOT_ALL, torch.float32)
        self.xchg = view(_lib.R_XCHG, torch.float32)  # dual backward: this rank's 4 b row statistics
        self.xall = view(_lib.R_XALL, torch.float32)  # ... all_gathered (alias at N = 1)
        self.pending_host = None  # (d_image, d_text, h_image, h_text) of a row-block step (dual fixup refresh)
        self.fixed_rows = 0       # rows the last step's dual fixup recomputed (set by the status read)
        status_all = view(_lib.R_STATUS, torch.uint8)
        status_all.zero_()  # the streamed forward's wave flags start below every epoch
        self.status = status_all[:24]
        self.feat = view(_lib.R_FEAT, torch.bfloat16).view(2, B, self.Dp)
        self.h2d_epoch = 0
        self.status_host = torch.empty(24, dtype=torch.uint8, pin_memory=True)
        self.waves = _lib.forward_waves(B, D, world, rank)
        self.pairs = torch.cuda.get_device_properties(device).multi_processor_count // 2  # persistent CTA pairs
        self._copy_stream = None
        self._gather_stream = None
        self._h2d_stream = None
        self._wave_stream = None
        self._pack_stream = None
        self._peer = None
        self._peer_group = None
        self.last_event = None   # end of the last enqueued use (cross-stream ordering, _enter)
        self.last_stream = None
        self.used = 0

    def peer_window(self, endpoint) -> "_peer.PeerWindow":
        """This rank's peer-transport window (created, and exchanged with the peers, on first use)."""
        group = getattr(endpoint, "group", None)
        if self._peer is not None and (self._peer_group is not group
                                       or self._peer.nbytes != _peer.window_bytes(self.B, self.D, self.world, self.rank)):
            self.close()  # a new group, or the backward mode changed the window layout: new windows
        if self._peer is None:
            self._peer = _peer.PeerWindow(endpoint, self.B, self.D, self.world, self.rank)
            self._peer_group = group
        return self._peer

    def close(self) -> None:
        if self._peer is not None:
            torch.cuda.synchronize(self.device)
            self._peer.close()
            self._peer = None

    def gather_stream(self) -> "torch.cuda.Stream":
        """Copy stream of the streamed peer all-gather (N > 1)."""
        if self._gather_stream is None:
            self._gather_stream = torch.cuda.Stream(self.device)
        return self._gather_stream

    def copy_stream(self) -> "torch.cuda.Stream":
        """Side stream for the pipelined device->host gradient copies (created on first use)."""
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(self.device)
        return self._copy_stream

    def pack_stream(self) -> "torch.cuda.Stream":
        """Stream of the wavefront forward's per-chunk packs (all in order on one stream)."""
        if self._pack_stream is None:
            self._pack_stream = torch.cuda.Stream(self.device)
        return self._pack_stream

    def h2d_streams(self):
        """(host->device copy stream, extra compute streams) of the wavefront forward: waves
        rotate over the current stream and these, so a wave's tail overlaps the next ones."""
        if self._h2d_stream is None:
            self._h2d_stream = torch.cuda.Stream(self.device)
            self._wave_stream = (torch.cuda.Stream(self.device), torch.cuda.Stream(self.device))
        return self._h2d_stream, self._wave_stream

    @property
    def args(self):
        return (self.ptr, self.B, self.D, self.world, self.rank)


# Plans are cached per (geometry, device, workspace size) -- not per thread, so fresh rank threads
# (run_ranks, a user's verify loop) reuse the workspace of the same rank/geometry.  The workspace
# size is part of the key because it follows the geometry the library computes right now.  The
# cache is bounded in bytes (least recently used plans are released first) and a plan used from
# a different stream than its last user first waits for that user's work (``_enter``).
_plans = {}
_plans_lock = threading.Lock()
_plan_clock = [0]


def _cache_cap(device: torch.device) -> int:
    env = os.environ.get("DISCO_PLAN_CACHE_BYTES")
    if env:
        return int(float(env))
    return int(0.6 * torch.cuda.get_device_properties(device).total_memory)


def _release(plan: Plan) -> None:
    if plan.last_event is not None:
        plan.last_event.synchronize()
    plan.close()


def get_plan(B: int, D: int, world: int, rank: int, device: torch.device) -> Plan:
    nbytes = _lib.workspace_bytes(B, D, world, rank)
    key = (B, D, world, rank, device.index, nbytes)
    with _plans_lock:
        _plan_clock[0] += 1
        plan = _plans.get(key)
        if plan is None:
            cap = _cache_cap(device)
            held = sum(p.ws.numel() for k, p in _plans.items() if k[4] == device.index)
            for k in sorted((k for k in _plans if k[4] == device.index), key=lambda k: _plans[k].used):
                if held + nbytes <= cap:
                    break
                victim = _plans.pop(k)
                held -= victim.ws.numel()
                _release(victim)
            plan = _plans[key] = Plan(B, D, world, rank, device)
        plan.used = _plan_clock[0]
        return plan


def cached_plans() -> int:
    """Number of cached workspaces (tests: the cache must not grow with rank threads)."""
    with _plans_lock:
        return len(_plans)


def clear_plans() -> None:
    with _plans_lock:
        for plan in _plans.values():
            _release(plan)
        _plans.clear()


def _enter(plan: Plan, stream) -> None:
    """Order this use of the plan's workspace after its previous user's work on another stream."""
    if plan.last_event is not None and plan.last_stream != stream.cuda_stream:
        stream.wait_event(plan.last_event)


def _leave(plan: Plan, stream) -> None:
    ev = torch.cuda.Event()
    ev.record(stream)
    plan.last_event, plan.last_stream = ev, stream.cuda_stream


# ---------------------------------------------------------------------------
# Input / output staging
# ---------------------------------------------------------------------------
def _default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the DisCo B200 path needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stage(x, device):
    """Return (device tensor, origin) for a numpy array or torch tensor; 2-D, unit column stride."""
    origin = "cuda"
    if isinstance(x, np.ndarray):
        origin = ("numpy", x.dtype)
        if x.ndim != 2:
            raise ShapeError(f"expected a 2-D matrix, got ndim={x.ndim}")
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"unsupported feature container {type(x)!r}")
    if x.dim() != 2:
        raise ShapeError(f"expected a 2-D matrix, got ndim={x.dim()}")
    if x.dtype not in _TORCH_DTYPE_CODE:
        x = x.to(torch.float32)
    if not x.is_cuda:
        if origin == "cuda":
            origin = "cpu"
        x = x.to(device, non_blocking=x.is_pinned())
    if x.stride(1) != 1 or (x.shape[0] > 1 and x.stride(0) < x.shape[1]):
        x = x.contiguous()
    return x, origin


def _on_host(x) -> bool:
    return isinstance(x, np.ndarray) or (isinstance(x, torch.Tensor) and not x.is_cuda)


def _host_tensor(x):
    """(row-contiguous CPU tensor, origin) for the H2D-pipelined path; same checks as _stage."""
    origin = "cpu"
    if isinstance(x, np.ndarray):
        origin = ("numpy", x.dtype)
        if x.ndim != 2:
            raise ShapeError(f"expected a 2-D matrix, got ndim={x.ndim}")
        x = torch.from_numpy(np.ascontiguousarray(x))
    if x.dim() != 2:
        raise ShapeError(f"expected a 2-D matrix, got ndim={x.dim()}")
    if x.dtype not in _TORCH_DTYPE_CODE:
        x = x.to(torch.float32)
    return x.contiguous(), origin


def _unstage_async(t: torch.Tensor, origin):
    """Start the device->host copy of an output into pinned memory (no sync)."""
    if origin == "cuda":
        return t
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t, non_blocking=True)
    return host


def _unstage_finish(h: torch.Tensor, origin):
    """After the stream synchronised: hand the host copy out in the caller's container."""
    if origin == "cuda" or origin == "cpu":
        return h
    _, dtype = origin
    out = h.numpy()
    return out.astype(dtype) if np.issubdtype(dtype, np.floating) and out.dtype != dtype else out


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _read_status(plan: Plan, with_dlogit: bool = False):
    plan.status_host.copy_(plan.status, non_blocking=True)
    torch.cuda.current_stream(plan.device).synchronize()
    raw = plan.status_host.numpy()
    loss = float(raw[:8].view(np.float64)[0])
    flags = int(raw[8:12].view(np.int32)[0])
    plan.fixed_rows = int(raw[12:16].view(np.int32)[0])  # dual backward rows recomputed exactly
    if with_dlogit:
        return loss, flags, float(raw[16:24].view(np.float64)[0])
    return loss, flags


def _raise_on_flags(flags: int) -> None:
    if flags & 1:
        raise ValueError("matmul result contains non-finite entries (non-finite input features)")
    if flags & 2:
        raise ValueError("cross-entropy logits contains non-finite entries")
    if flags & 4:
        raise ValueError("gradient contribution contains non-finite entries")
    if flags & 16:
        raise RuntimeError("streamed forward: a host->device chunk never landed (wave flag timeout)")
    if flags & 8:
        raise CollectiveTimeoutError(
            f"peer transport: gradient slabs did not arrive within {_peer.PEER_TIMEOUT_S:g}s")


def _check_t(t) -> float:
    t = float(t)
    if not t > 0 or not np.isfinite(t):
        raise DomainError(f"temperature must be positive, got {t}")
    return t


# ---------------------------------------------------------------------------
# Public entry points
# ---------------------------------------------------------------------------
def local_loss_and_grads(layout: ShardLayout, I_gathered, T_gathered, t: float, *,
                         loss_counters: Counters | None = None,
                         exchange_counters: Counters | None = None,
                         flip_cross_rank_sign: bool = False) -> LocalGradContribution:
    """One rank's loss rows and full-size gradient contribution (shard.py:98-166).

    ``I_gathered`` / ``T_gathered`` are the B x D gathered features (numpy or
    torch).  Returns B x D fp32 contributions whose rank-mean is the full-batch
    gradient, and the rank's local loss (mean of its two CE halves).
    """
    if t <= 0:
        raise DomainError(f"temperature must be positive, got {t}")
    if tuple(I_gathered.shape) != tuple(T_gathered.shape):
        raise ShapeError(
            f"gathered shapes disagree: {tuple(I_gathered.shape)} vs {tuple(T_gathered.shape)}")
    if I_gathered.shape[0] != layout.global_batch:
        raise LayoutError(
            f"gathered matrices have {I_gathered.shape[0]} rows, layout "
            f"expects {layout.global_batch}")
    if len(I_gathered.shape) != 2:
        raise ShapeError("gathered features must be 2-D")
    t = _check_t(t)
    device = _default_device()
    Ig, origin = _stage(I_gathered, device)
    Tg, _ = _stage(T_gathered, device)
    N, B, D, n = layout.world_size, layout.global_batch, Ig.shape[1], layout.rank
    b = layout.local_batch
    plan = get_plan(B, D, N, n, device)
    cur_stream = torch.cuda.current_stream(device)
    _enter(plan, cur_stream)
    st = cur_stream.cuda_stream
    code = _TORCH_DTYPE_CODE[Ig.dtype]
    if Tg.dtype != Ig.dtype:
        Tg = Tg.to(Ig.dtype)
    per_rank = 2 * b * plan.Dp
    for src in range(N):
        Is, Ts = Ig[src * b:(src + 1) * b], Tg[src * b:(src + 1) * b]
        _lib.call("disco_b200_pack", *plan.args, Is.data_ptr(), Ts.data_ptr(), Is.stride(0),
                  Ts.stride(0), code, int(src == 0), st)
        if N > 1:
            plan.gather[src * per_rank:(src + 1) * per_rank].copy_(plan.pack)
    _lib.call("disco_b200_forward", *plan.args, t, st)
    _lib.call("disco_b200_backward_grad", *plan.args, t, st)
    _lib.call("disco_b200_backward_cross", *plan.args, st)
    _lib.call("disco_b200_backward_intra", *plan.args, st)
    d_image = torch.empty((B, D), dtype=torch.float32, device=device)
    d_text = torch.empty((B, D), dtype=torch.float32, device=device)
    _lib.call("disco_b200_contribution", *plan.args, t, int(bool(flip_cross_rank_sign)),
              d_image.data_ptr(), d_text.data_ptr(), D, st)
    _lib.call("disco_b200_loss", *plan.args, 1, st)
    _leave(plan, cur_stream)
    h_image, h_text = _unstage_async(d_image, origin), _unstage_async(d_text, origin)
    loss, flags = _read_status(plan)
    _raise_on_flags(flags)
    _account_loss_scope(loss_counters, exchange_counters, b, B, D)
    return LocalGradContribution(_unstage_finish(h_image, origin), _unstage_finish(h_text, origin), loss)


def _account_loss_scope(loss_counters, exchange_counters, b, B, D) -> None:
    """The reference's analytic accounting of local_loss_and_grads (shard.py:133-156)."""
    if loss_counters is not None:
        with tracking(loss_counters):
            loss_counters.add_flops(4 * b * B * D)
        loss_counters.alloc(2 * b * B)
    if exchange_counters is not None:
        exchange_counters.add_flops(8 * b * B * D)
        exchange_counters.alloc(2 * B * D)
    if loss_counters is not None:
        loss_counters.release(2 * b * B)


# Fractions of the 256-row tiles per output row block of the pipelined backward: shrinking by
# ~0.8 per block (32, 25, 20, 16, 12, 10, 8, 5 of 128 tiles), so each block's device->host copy
# (19 us/tile) fits under the next block's GEMMs (24 us/tile) and the exposed tail is the last
# 5 tiles.  Measured with tools/e2e_ab.py against quarters-then-eighths: -0.09 ms e2e; faster
# shrinking (more, smaller launches) or intra-ahead schedules measured slower.
ROW_BLOCK_FRACTIONS = (0.25, 0.1953125, 0.15625, 0.125, 0.09375, 0.078125, 0.0625, 0.0390625)


def fused_row_blocks(b: int, pairs: int, units_per_tile: int = 4):
    """Row blocks for the single-rank dual backward (disco_b200_path_info PATH_DUAL): its units
    are long (a K half of all B columns) and only ``units_per_tile`` per 256-row tile, so every
    block is one whole wave of the ``pairs`` CTA pairs.  A wave's gradients (~19 MB at D = 512)
    are produced faster than PCIe drains them, so the device->host copy never waits after the
    first block: the step is bounded by the copy (tools/e2e_timeline.py)."""
    tiles = (b + 255) // 256
    w1 = max(1, pairs // units_per_tile)  # tiles per wave
    cuts = list(range(0, tiles, w1)) + [tiles]
    return [(min(256 * lo, b), min(256 * hi, b)) for lo, hi in zip(cuts, cuts[1:])]


def row_blocks(b: int, fractions=None):
    """Output row blocks of the single-rank pipelined backward (fractions of the 256-row tiles,
    ROW_BLOCK_FRACTIONS by default; one block for small b)."""
    fractions = fractions or ROW_BLOCK_FRACTIONS
    tiles = (b + 255) // 256
    if tiles < 8:
        return [(0, b)]
    cuts, acc = [0], 0.0
    for f in fractions[:-1]:
        acc += f
        c = max(cuts[-1] + 1, round(acc * tiles))
        if c < tiles:
            cuts.append(c)
    cuts.append(tiles)
    return [(min(256 * lo, b), min(256 * hi, b)) for lo, hi in zip(cuts, cuts[1:])]


def _pipelined_pack_forward(plan: Plan, I_host: torch.Tensor, T_host: torch.Tensor, t: float) -> None:
    """Single rank, host features: H2D copy in canonical row chunks on a copy stream; as chunk k
    lands its rows are packed and forward wave k runs (the logit units that chunk k completes),
    alternating between two compute streams so one wave's tail overlaps the next.  Bit-identical
    to pack + disco_b200_forward (the waves partition the units; every unit is unchanged)."""
    device = plan.device
    cur = torch.cuda.current_stream(device)
    h2d, side = plan.h2d_streams()
    b, D = I_host.shape
    code = _TORCH_DTYPE_CODE[I_host.dtype]
    I_dev = torch.empty(I_host.shape, dtype=I_host.dtype, device=device)
    T_dev = torch.empty(T_host.shape, dtype=T_host.dtype, device=device)
    # status reset before any wave can raise a flag, on the stream every other stream follows
    _lib.call("disco_b200_pack_rows", *plan.args, I_dev.data_ptr(), T_dev.data_ptr(), D, D, code, 1, 0, 0,
              cur.cuda_stream)
    h2d.wait_stream(cur)
    for s in side:
        s.wait_stream(cur)
    rows = b // plan.waves
    streams = (cur,) + side
    pack = plan.pack_stream()
    pack.wait_stream(cur)
    for k in range(plan.waves):  # enqueue copy k, then its wave, so wave 0 launches early
        sl = slice(k * rows, (k + 1) * rows)
        with torch.cuda.stream(h2d):
            I_dev[sl].copy_(I_host[sl], non_blocking=True)
            T_dev[sl].copy_(T_host[sl], non_blocking=True)
        landed = torch.cuda.Event()
        landed.record(h2d)
        # wave k reads the packed rows of chunks 0..k: every pack runs in order on ONE stream, so
        # the event after pack k covers all earlier packs (waves rotate over three streams)
        pack.wait_event(landed)
        _lib.call("disco_b200_pack_rows", *plan.args, I_dev.data_ptr(), T_dev.data_ptr(), D, D, code, 0,
                  k * rows, (k + 1) * rows, pack.cuda_stream)
        packed = torch.cuda.Event()
        packed.record(pack)
        s = streams[k % len(streams)]
        s.wait_event(packed)
        _lib.call("disco_b200_forward_wave", *plan.args, t, k, s.cuda_stream)
    for s in side + (pack,):
        cur.wait_stream(s)
    for x in (I_dev, T_dev):
        x.record_stream(h2d)
        for s in side + (pack,):
            x.record_stream(s)
    _lib.call("disco_b200_forward_finish", *plan.args, cur.cuda_stream)


# host bf16 features with D % 64 == 0: one persistent, flag-gated logits launch (streamed forward)
STREAMED_FORWARD = True
H2D_TIMEOUT_S = 30.0
# split host-buffer schedule (split_schedule): env DISCO_SPLIT=0 selects the one-launch forward
SPLIT_SCHEDULE = os.environ.get("DISCO_SPLIT", "1") not in ("", "0")


def _streamed_forward(plan: Plan, I_host: torch.Tensor, T_host: torch.Tensor, t: float, k0=None) -> None:
    """Single rank, host bf16 features: chunk k's rows are copied straight into the forward
    operands (DISCO_R_FEAT) on a copy stream, each followed by a stream write of the wave flag;
    ONE persistent logits kernel walks the waves in order, its producers waiting on each flag.
    Bit-identical to pack + disco_b200_forward.  ``k0`` (split schedule): the kernel runs all of
    direction 1 and direction 0 only for waves < k0 (the rest: ``_split_backward``)."""
    device = plan.device
    cur = torch.cuda.current_stream(device)
    h2d, _ = plan.h2d_streams()
    b, D = I_host.shape
    feat = plan.feat
    # status reset, ordered before everything of this step (no rows are packed: 0..0)
    _lib.call("disco_b200_pack_rows", *plan.args, feat.data_ptr(), feat.data_ptr(), D, D, _lib.BF16, 1, 0, 0,
              cur.cuda_stream)
    h2d.wait_stream(cur)  # the previous step is done with FEAT
    plan.h2d_epoch = (plan.h2d_epoch + 1) & 0x7FFFFFFF or 1
    epoch = plan.h2d_epoch
    # every copy and wave signal is enqueued (one native call) BEFORE the kernel that waits on them
    _lib.call("disco_b200_h2d_streamed", *plan.args, I_host.data_ptr(), T_host.data_ptr(), epoch, h2d.cuda_stream)
    plan.h2d_keepalive = (I_host, T_host)  # raw-pointer copies: keep the host rows alive past this step
    if k0 is None:
        _lib.call("disco_b200_forward_streamed", *plan.args, t, epoch, H2D_TIMEOUT_S, cur.cuda_stream)
    else:
        _lib.call("disco_b200_forward_streamed_split", *plan.args, t, epoch, H2D_TIMEOUT_S, int(k0), cur.cuda_stream)
    cur.wait_stream(h2d)


def split_schedule(plan: Plan):
    """(k0, row blocks) of the split host-buffer schedule, or None when it does not apply.

    Direction 1 runs inside the H2D wavefront together with direction 0 of the first k0 waves
    (about the work the copies leave room for); the rest of direction 0 then runs row block by
    row block, each followed by that block's d_image backward and its copy to the host, so the
    device->host stream starts about one block after the wavefront instead of after the whole
    forward.  Blocks hold whole waves and ~one CTA-pair wave of backward units (two K halves per
    256-row tile of ONE direction)."""
    if not SPLIT_SCHEDULE or plan.world != 1 or plan.waves < 4:
        return None
    nw = plan.waves
    k0 = int(os.environ.get("DISCO_SPLIT_K0", "-1"))
    if k0 < 0:
        k0 = (3 * nw) // 4
    k0 = max(0, min(nw, k0))
    rows_per_wave = plan.b // nw
    if rows_per_wave % 256:
        return None
    tiles_per_block = max(1, plan.pairs // 2)                  # 2 K halves per 256-row tile, one direction
    waves_per_block = max(1, (tiles_per_block * 256) // rows_per_wave)
    cuts = list(range(0, nw, waves_per_block)) + [nw]
    return k0, [(w0 * rows_per_wave, w1 * rows_per_wave) for w0, w1 in zip(cuts, cuts[1:])]


def _split_backward(plan: Plan, t: float, flip: int, k0: int, blocks, d_image, d_text, host_out) -> None:
    """Second half of the split schedule (after ``_streamed_forward(..., k0)``): direction 0's
    remaining units per row block, its statistics, its d_image backward + combine and the block's
    copy to the host; then, with every row's statistics known, the d_text blocks.  Each unit,
    tile, K order and reduction is the one of the one-launch path: the same bits."""
    device, b, D = plan.device, plan.b, plan.D
    st = torch.cuda.current_stream(device).cuda_stream
    nw = plan.waves
    rows_per_wave = b // nw
    cs = plan.copy_stream()
    cur = torch.cuda.current_stream(device)
    h_image, h_text = host_out
    _lib.call("disco_b200_dual_prep_dir", *plan.args, 0, flip, st)
    for r0, r1 in blocks:
        w0, w1 = r0 // rows_per_wave, r1 // rows_per_wave
        if w0 < k0:  # waves already in the wavefront's direction-0 share: only chunks >= k0 are left
            e = min(w1, k0) * rows_per_wave
            if k0 < nw:
                _lib.call("disco_b200_forward_rect", *plan.args, t, 0, r0, e, k0, nw, st)
            if e < r1:
                _lib.call("disco_b200_forward_rect", *plan.args, t, 0, e, r1, 0, nw, st)
        else:
            _lib.call("disco_b200_forward_rect", *plan.args, t, 0, r0, r1, 0, nw, st)
        _lib.call("disco_b200_stats_rows", *plan.args, 0, r0, r1, st)
        _lib.call("disco_b200_backward_dual_dir", *plan.args, 0, r0, r1, st)
        _lib.call("disco_b200_combine_dual_dir", *plan.args, 0, t, r0, r1, d_image.data_ptr(), d_text.data_ptr(), D, st)
        cs.wait_stream(cur)
        with torch.cuda.stream(cs):
            h_image[r0:r1].copy_(d_image[r0:r1], non_blocking=True)
    _lib.call("disco_b200_dual_prep_dir", *plan.args, 1, flip, st)
    for r0, r1 in blocks:
        _lib.call("disco_b200_backward_dual_dir", *plan.args, 1, r0, r1, st)
        _lib.call("disco_b200_combine_dual_dir", *plan.args, 1, t, r0, r1, d_image.data_ptr(), d_text.data_ptr(), D, st)
        cs.wait_stream(cur)
        with torch.cuda.stream(cs):
            h_text[r0:r1].copy_(d_text[r0:r1], non_blocking=True)
    d_image.record_stream(cs)
    d_text.record_stream(cs)
    plan.pending_host = (d_image, d_text, h_image, h_text)
    _lib.call("disco_b200_dual_fixup", *plan.args, t, flip, d_image.data_ptr(), d_text.data_ptr(), D, st)
    _lib.call("disco_b200_loss", *plan.args, 2, st)


def host_pipelined(world: int, B: int, D: int, rank: int = 0) -> bool:
    """True when disco_step_async overlaps the H2D copy of host features with the forward."""
    return world == 1 and _lib.forward_waves(B, D, world, rank) > 0


def disco_step_async(endpoint, local_I, local_T, t: float, *, flip_cross_rank_sign: bool = False,
                     host_out=None, l2norm=None):
    """Launch one rank's DisCo fwd+bwd without any host synchronisation.

    Inputs are CUDA tensors (b x D), or, on a single rank with a wavefront-capable
    shape (``host_pipelined``), CPU tensors (pinned for a fully asynchronous copy):
    their H2D copy then overlaps the forward GEMMs chunk by chunk.  Returns
    (d_image, d_text, plan); the global loss and the non-finite flags are read
    later with ``finish_status(plan)``.  ``disco_step`` is this plus that read-back.

    ``host_out`` = (h_image, h_text) pinned host tensors (single rank): the
    backward then runs in output row blocks and each block's gradients are
    copied to the host on ``plan.copy_stream`` while the next block computes
    (wait on that stream, or call ``finish_status``, before reading them).

    ``l2norm`` = (raw_I, raw_T, dx_I, dx_T, norm_flags), device fp32 (the two-tower caller,
    towers.py:244-280): the features are l2_normalize_rows(raw); the combine then also writes
    dx = l2_normalize_rows_backward(raw, d) into dx_I / dx_T (fused in its epilogue on the dual
    path, the separate kernel otherwise; bitwise equal either way) and ORs bit0 (non-finite dx)
    / bit1 (norm < 1e-12) into the int32 ``norm_flags``.
    """
    N, n = endpoint.world_size, endpoint.rank
    _check_step_inputs(local_I, local_T)
    b, D = local_I.shape
    B = b * N
    on_host = not local_I.is_cuda
    device = _default_device() if on_host else local_I.device
    plan = get_plan(B, D, N, n, device)
    cur_stream = torch.cuda.current_stream(device)
    _enter(plan, cur_stream)
    st = cur_stream.cuda_stream
    pw = None  # peer window of this step (N > 1 with the peer transport)
    split = None  # (k0, row blocks) of the split host-buffer schedule
    if on_host:
        if N != 1 or plan.waves == 0 or local_T.is_cuda:
            raise ValueError("host (CPU) features need a single rank and a wavefront shape; "
                             "stage them to the device first")
        if (STREAMED_FORWARD and local_I.dtype == torch.bfloat16 and local_T.dtype == torch.bfloat16
                and D == plan.Dp and local_I.is_contiguous() and local_T.is_contiguous()
                and local_I.is_pinned() and local_T.is_pinned()):
            if host_out is not None and l2norm is None and _lib.path_info(B, D, N, n) & _lib.PATH_DUAL:
                split = split_schedule(plan)
            _streamed_forward(plan, local_I.contiguous(), local_T.contiguous(), t,
                              split[0] if split is not None else None)
        else:
            _pipelined_pack_forward(plan, local_I.contiguous(), local_T.contiguous(), t)
    else:
        code = _TORCH_DTYPE_CODE[local_I.dtype]
        _lib.call("disco_b200_pack", *plan.args, local_I.data_ptr(), local_T.data_ptr(),
                  local_I.stride(0), local_T.stride(0), code, 1, st)
        if N > 1 and _peer.enabled(endpoint) and _peer.supported(B, D, N, n):
            # peer transport: every rank reads the others' packed rows from their NVLink-mapped
            # windows straight into its operand layouts (all_gather + unpack in one kernel)
            try:
                pw = plan.peer_window(endpoint)
            except _peer.PeerUnavailable:
                endpoint.peer = False  # collective decision: every rank falls back to the NCCL exchange
                pw = None
        if pw is not None:
            epoch, parity = pw.next_step()
            _lib.call("disco_b200_peer_publish", *plan.args, pw.bases, parity, epoch, st)
            _peer.in_process_fence(endpoint, cur_stream)
            if _peer.streamed_gather(endpoint, B, N):
                # copy-engine pulls gated by the peers' pack-ready flags, enqueued BEFORE the one
                # persistent logits launch that consumes them column wave by column wave
                cur = torch.cuda.current_stream(device)
                gs = plan.gather_stream()
                gs.wait_stream(cur)
                _lib.call("disco_b200_peer_gather_streamed", *plan.args, pw.bases, parity, epoch, gs.cuda_stream)
                _lib.call("disco_b200_forward_peer_streamed", *plan.args, t, epoch, _peer.PEER_TIMEOUT_S, st)
                cur.wait_stream(gs)
            else:
                _lib.call("disco_b200_peer_gather", *plan.args, pw.bases, parity, epoch, _peer.PEER_TIMEOUT_S, st)
                _lib.call("disco_b200_forward_gathered", *plan.args, t, st)
        elif N > 1:
            endpoint.all_gather_into(plan.gather, plan.pack)
            _lib.call("disco_b200_forward", *plan.args, t, st)
        else:
            _lib.call("disco_b200_forward", *plan.args, t, st)
    d_image = torch.empty((b, D), dtype=torch.float32, device=device)
    d_text = torch.empty((b, D), dtype=torch.float32, device=device)
    flip = int(bool(flip_cross_rank_sign))
    if l2norm is not None:
        _check_l2norm_args(l2norm, b, D, device)
    fused = l2norm is not None and host_out is None and bool(_lib.path_info(B, D, N, n) & _lib.PATH_DUAL)
    if split is not None:
        _split_backward(plan, t, flip, split[0], split[1], d_image, d_text, host_out)
    elif _lib.path_info(B, D, N, n) & _lib.PATH_DUAL:
        _dual_backward(endpoint, plan, t, flip, d_image, d_text, host_out, l2norm if fused else None)
    else:
        _exchange_backward(endpoint, plan, t, flip, d_image, d_text, host_out, pw,
                           parity if pw is not None else 0, epoch if pw is not None else 0)
    if l2norm is not None and not fused:
        raw_I, raw_T, dx_I, dx_T, nf = l2norm
        for raw, d, dx in ((raw_I, d_image, dx_I), (raw_T, d_text, dx_T)):
            _lib.call("disco_b200_l2norm_rows_backward", raw.data_ptr(), raw.stride(0), d.data_ptr(), d.stride(0),
                      b, D, dx.data_ptr(), dx.stride(0), nf.data_ptr(), st)
    _leave(plan, cur_stream)
    return d_image, d_text, plan


def _check_l2norm_args(l2norm, b: int, D: int, device) -> None:
    """The fused normalisation backward writes through raw pointers: reject anything that is not
    (b x D fp32 row-major CUDA tensors on the plan's device, an int32 flag word) before a launch."""
    if len(l2norm) != 5:
        raise TypeError("l2norm must be (raw_I, raw_T, dx_I, dx_T, norm_flags)")
    *mats, nf = l2norm
    for m in mats:
        if not (isinstance(m, torch.Tensor) and m.is_cuda and m.device == device and m.dtype == torch.float32
                and m.dim() == 2 and tuple(m.shape) == (b, D) and m.stride(1) == 1 and m.stride(0) >= D):
            raise ShapeError(f"l2norm tensors must be ({b}, {D}) float32 row-major on {device}")
    if not (isinstance(nf, torch.Tensor) and nf.is_cuda and nf.device == device and nf.dtype == torch.int32
            and nf.numel() >= 1):
        raise ShapeError("l2norm norm_flags must be an int32 CUDA tensor")


def _dual_backward(endpoint, plan: Plan, t: float, flip: int, d_image, d_text, host_out, l2norm=None) -> None:
    """The dual backward (disco_b200_path_info PATH_DUAL): all_gather the 4 b row statistics, then
    one GEMM per gradient over the rank's own E block (H = G_d + G_d'^T), the combine with the
    fp32 label term, the exact recompute of any flagged rows, and the loss from the gathered ce.
    Replaces the reference's all_reduce(AVG) + slice (shard.py:199-208): no gradient exchange."""
    device, b, D, N = plan.device, plan.b, plan.D, plan.world
    st = torch.cuda.current_stream(device).cuda_stream
    if N > 1:
        endpoint.all_gather_into(plan.xall, plan.xchg)
    _lib.call("disco_b200_dual_prep", *plan.args, flip, st)
    if host_out is not None:  # rank-local row blocks at every N: each block's copy overlaps the next
        cs = plan.copy_stream()
        cur = torch.cuda.current_stream(device)
        h_image, h_text = host_out
        for r0, r1 in fused_row_blocks(b, plan.pairs):
            _lib.call("disco_b200_backward_dual", *plan.args, r0, r1, st)
            _lib.call("disco_b200_combine_dual", *plan.args, t, r0, r1, d_image.data_ptr(), d_text.data_ptr(), D, st)
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                h_image[r0:r1].copy_(d_image[r0:r1], non_blocking=True)
                h_text[r0:r1].copy_(d_text[r0:r1], non_blocking=True)
        d_image.record_stream(cs)
        d_text.record_stream(cs)
        plan.pending_host = (d_image, d_text, h_image, h_text)
    elif l2norm is not None:  # two-tower step: the normalisation backward fused into the combine
        raw_I, raw_T, dx_I, dx_T, nf = l2norm
        _lib.call("disco_b200_backward_dual", *plan.args, 0, b, st)
        _lib.call("disco_b200_finish_dual_l2norm", *plan.args, t, flip, raw_I.data_ptr(), raw_I.stride(0),
                  raw_T.data_ptr(), raw_T.stride(0), d_image.data_ptr(), d_text.data_ptr(), D, dx_I.data_ptr(),
                  dx_T.data_ptr(), dx_I.stride(0), nf.data_ptr(), st)
    else:
        _lib.call("disco_b200_backward_dual", *plan.args, 0, b, st)
        _lib.call("disco_b200_combine_dual", *plan.args, t, 0, b, d_image.data_ptr(), d_text.data_ptr(), D, st)
    if l2norm is None or host_out is not None:
        _lib.call("disco_b200_dual_fixup", *plan.args, t, flip, d_image.data_ptr(), d_text.data_ptr(), D, st)
    _lib.call("disco_b200_loss", *plan.args, 2, st)


def _exchange_backward(endpoint, plan: Plan, t: float, flip: int, d_image, d_text, host_out, pw, parity: int,
                       epoch: int) -> None:
    """The exchange backward (DISCO_BACKWARD=exchange, or shapes without stored E): intra and
    cross GEMMs, then the reference's all_reduce(AVG) + slice as a reduce-scatter -- over the peer
    transport (cross tiles pushed from the GEMM epilogue) or an NCCL all_to_all."""
    device, b, D, N = plan.device, plan.b, plan.D, plan.world
    st = torch.cuda.current_stream(device).cuda_stream
    _lib.call("disco_b200_backward_grad", *plan.args, t, st)
    if pw is not None:
        # the fused backward GEMM pushes each cross tile to its owner over NVLink
        _lib.call("disco_b200_backward_peer", *plan.args, pw.bases, parity, epoch, st)
        _peer.in_process_fence(endpoint, torch.cuda.current_stream(device))
    elif N > 1:
        # cross first, so the slab exchange overlaps the intra GEMM
        _lib.call("disco_b200_backward_cross", *plan.args, st)
        work = endpoint.all_to_all_into(plan.recv, plan.send, async_op=True)
        _lib.call("disco_b200_backward_intra", *plan.args, st)
        work.wait()
    if N == 1 and host_out is not None:
        cs = plan.copy_stream()
        cur = torch.cuda.current_stream(device)
        h_image, h_text = host_out
        for r0, r1 in row_blocks(b):
            _lib.call("disco_b200_backward_rows", *plan.args, r0, r1, st)
            _lib.call("disco_b200_combine_rows", *plan.args, t, flip, r0, r1,
                      d_image.data_ptr(), d_text.data_ptr(), D, st)
            cs.wait_stream(cur)
            with torch.cuda.stream(cs):
                h_image[r0:r1].copy_(d_image[r0:r1], non_blocking=True)
                h_text[r0:r1].copy_(d_text[r0:r1], non_blocking=True)
        d_image.record_stream(cs)
        d_text.record_stream(cs)
    elif pw is not None:
        _lib.call("disco_b200_combine_peer", *plan.args, t, flip, pw.base, parity, epoch, _peer.PEER_TIMEOUT_S,
                  d_image.data_ptr(), d_text.data_ptr(), D, st)
    else:
        if N == 1:
            _lib.call("disco_b200_backward_fused", *plan.args, st)
        _lib.call("disco_b200_combine", *plan.args, t, flip, d_image.data_ptr(), d_text.data_ptr(), D, st)
    if pw is not None:  # every rank's ce arrived with its slabs (covered by the combine's wait)
        _lib.call("disco_b200_loss_peer", *plan.args, pw.base, parity, st)
    else:
        if N > 1:
            endpoint.all_gather_into(plan.ce_all, plan.ce)
        _lib.call("disco_b200_loss", *plan.args, 0, st)


def _check_step_inputs(local_I, local_T) -> None:
    """What the kernels assume of ``disco_step_async``'s inputs (the checks ``disco_step`` gets
    from ``_stage``): tensors, 2-D, equal shapes and dtypes, a supported dtype, unit column
    stride with rows at least D apart, both on the same device.  Raises ShapeError / TypeError
    before any launch, so a bad view cannot make a kernel read out of bounds."""
    for x in (local_I, local_T):
        if not isinstance(x, torch.Tensor):
            raise TypeError(f"disco_step_async takes torch tensors, got {type(x)!r}")
        if x.dim() != 2:
            raise ShapeError(f"expected a 2-D matrix, got ndim={x.dim()}")
    if tuple(local_I.shape) != tuple(local_T.shape):
        raise ShapeError(
            f"local feature shapes disagree: {tuple(local_I.shape)} vs {tuple(local_T.shape)}")
    if local_I.dtype != local_T.dtype:
        raise TypeError(f"feature dtypes disagree: {local_I.dtype} vs {local_T.dtype}")
    if local_I.dtype not in _TORCH_DTYPE_CODE:
        raise TypeError(f"unsupported feature dtype {local_I.dtype} (f32, bf16, f16, f64)")
    if local_I.device != local_T.device:
        raise ValueError(f"features on different devices: {local_I.device} vs {local_T.device}")
    if local_I.shape[0] == 0 or local_I.shape[1] == 0:
        raise ShapeError(f"empty feature matrix {tuple(local_I.shape)}")
    for x in (local_I, local_T):
        if x.stride(1) != 1 or (x.shape[0] > 1 and x.stride(0) < x.shape[1]):
            raise ShapeError(
                f"features need unit column stride and row stride >= D (got strides {tuple(x.stride())}); "
                "pass .contiguous()")


def finish_status(plan: Plan) -> float:
    loss, flags = _read_status(plan)
    if plan._copy_stream is not None:
        plan._copy_stream.synchronize()
    _refresh_host_rows(plan)
    _raise_on_flags(flags)
    return loss


def _refresh_host_rows(plan: Plan) -> None:
    """Row-block steps copy each block to the host as soon as it is combined; rows the dual
    fixup recomputed afterwards (plan.fixed_rows > 0, normally none) are copied again here."""
    pending, plan.pending_host = plan.pending_host, None
    if pending is not None and plan.fixed_rows > 0:
        d_image, d_text, h_image, h_text = pending
        h_image.copy_(d_image)
        h_text.copy_(d_text)


def logit_scale_grad_async(endpoint, plan: Plan, d_image, d_text, t: float) -> None:
    """Queue dL/dt after ``disco_step_async``: per-row
    <d, features> terms, all_gather across ranks (N > 1), fixed-order sum.  Read it
    with ``finish_status_with_dlogit``."""
    st = _stream_ptr(plan.device)
    _lib.call("disco_b200_logit_scale_rows", *plan.args, d_image.data_ptr(), d_text.data_ptr(),
              d_image.stride(0), st)
    if plan.world > 1:
        endpoint.all_gather_into(plan.rdot_all, plan.rdot)
    _lib.call("disco_b200_logit_scale_grad", *plan.args, t, st)


def finish_status_with_dlogit(plan: Plan):
    """(global loss, dL/dt) after ``logit_scale_grad_async``; raises on non-finite flags."""
    loss, flags, dlogit = _read_status(plan, with_dlogit=True)
    _raise_on_flags(flags)
    return loss, dlogit


def disco_step(endpoint, local_I, local_T, t: float, *, loss_counters: Counters | None = None,
               exchange_counters: Counters | None = None,
               flip_cross_rank_sign: bool = False):
    """One rank's share of the sharded loss step (shard.py:169-208).

    Returns (d_image_local, d_text_local, global_loss): fp32 b x D gradients of
    the full-batch loss for this rank's rows and the loss (identical on every
    rank).  ``endpoint`` is any object with the fabric protocol
    (``ProcessGroupEndpoint``, ``LocalEndpoint``) or None for world size 1.
    Outputs follow the inputs' container: numpy in -> numpy out (host copies
    included), CUDA tensors in -> CUDA tensors out.
    """
    if endpoint is None:
        endpoint = SingleEndpoint()
    if tuple(local_I.shape) != tuple(local_T.shape):
        raise ShapeError(
            f"local feature shapes disagree: {tuple(local_I.shape)} vs {tuple(local_T.shape)}")
    if exchange_counters is None:
        exchange_counters = Counters()
    layout = ShardLayout(world_size=endpoint.world_size,
                         global_batch=local_I.shape[0] * endpoint.world_size,
                         rank=endpoint.rank)
    t = _check_t(t)
    batch, dim = layout.global_batch, local_I.shape[1]
    device = _default_device()
    if endpoint.world_size == 1 and host_pipelined(1, batch, dim) and _on_host(local_I) and _on_host(local_T):
        I_dev, origin = _host_tensor(local_I)  # H2D happens inside, chunk by chunk
        T_dev, _ = _host_tensor(local_T)
    else:
        I_dev, origin = _stage(local_I, device)
        T_dev, _ = _stage(local_T, device)
    if T_dev.dtype != I_dev.dtype:
        T_dev = T_dev.to(I_dev.dtype)
    exchange_counters.alloc(2 * batch * dim)
    host_out = None
    # pipelined read-back (row blocks): single rank, or any N on the dual path (rank-local rows)
    if origin != "cuda" and (endpoint.world_size == 1
                             or _lib.path_info(batch, dim, endpoint.world_size, endpoint.rank) & _lib.PATH_DUAL):
        shape = (layout.local_batch, dim)
        host_out = (torch.empty(shape, dtype=torch.float32, pin_memory=True),
                    torch.empty(shape, dtype=torch.float32, pin_memory=True))
    d_image, d_text, plan = disco_step_async(endpoint, I_dev, T_dev, t,
                                             flip_cross_rank_sign=flip_cross_rank_sign, host_out=host_out)
    if host_out is not None:
        h_image, h_text = host_out
    else:
        h_image, h_text = _unstage_async(d_image, origin), _unstage_async(d_text, origin)
    loss = finish_status(plan)
    _account_loss_scope(loss_counters, exchange_counters, layout.local_batch, batch, dim)
    exchange_counters.alloc(batch * dim)
    exchange_counters.release(batch * dim)
    exchange_counters.alloc(batch * dim)
    exchange_counters.release(batch * dim)
    return _unstage_finish(h_image, origin), _unstage_finish(h_text, origin), loss
