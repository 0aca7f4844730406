"""Rank endpoints: the collective backend of the DisCo loss.

The reference simulates ranks as threads over an in-process fabric
(reference fabric.py:246-324).  Here a rank is a CUDA device and collectives
run over NCCL (NVLink 5 / NVSwitch on a B200 box) through torch.distributed.
Two endpoint kinds share one protocol:

* ``ProcessGroupEndpoint`` -- one process per GPU (torchrun), NCCL for CUDA
  tensors, gloo for CPU tensors (the multi-process CPU tests).
* ``run_ranks`` / ``LocalEndpoint`` -- N simulated ranks as threads of one
  process, all on the same device, with device-side copies as the transport.
  This is how the single-GPU tests check that results are bitwise identical
  across world sizes; it mirrors the reference's ``run_ranks``
  (fabric.py:291-324) in concurrent mode (the lockstep schedule explorer is a
  reference test harness and out of scope).

Protocol (reference-compatible methods first, fabric.py:257-275):
  rank, world_size
  all_gather(local) -> rank-order concatenation along dim 0
  all_reduce(buffer, op) -> elementwise SUM / AVG, accumulated in ascending rank order
  all_reduce_scalar(value, op) -> float
  barrier()
Fast paths used by ``disco_step`` (device tensors, preallocated outputs):
  all_gather_into(out, inp)            out = concat_r inp_r (flat, equal sizes)
  all_to_all_into(out, inp, async_op)  out[src block] = inp_src[dest block]
"""

import enum
import threading
import time

import torch
import torch.distributed as dist

from .errors import CollectiveContractError, CollectiveTimeoutError

DEFAULT_TIMEOUT = 300.0
LOCKSTEP, CONCURRENT = "lockstep", "concurrent"  # reference scheduler names (fabric.py); ranks run as threads


class ReduceOp(enum.Enum):
    SUM = "sum"
    AVG = "avg"


def _as_op(op) -> ReduceOp:
    if isinstance(op, ReduceOp):
        return op
    return ReduceOp(str(op).lower())


def _ordered_reduce(parts, op: ReduceOp):
    """Ascending-rank sum then one division for AVG (reference fabric.py:86-93)."""
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    if op is ReduceOp.AVG:
        acc /= len(parts)
    return acc


class _DoneWork:
    def wait(self):
        return True


class ProcessGroupEndpoint:
    """One rank's handle over a torch.distributed process group."""

    in_process = False

    def __init__(self, group=None, peer=None):
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialized")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world_size = dist.get_world_size(group)
        self.peer = peer  # None: env DISCO_PEER decides (peer.enabled)
        # gloo cannot move CUDA tensors: stage the device fast paths through host memory (tests)
        self._host_staged = dist.get_backend(group) != "nccl"

    def exchange(self, obj) -> list:
        """All ranks' picklable objects, in rank order (peer-window handles)."""
        out = [None] * self.world_size
        dist.all_gather_object(out, obj, group=self.group)
        return out

    # -- fast paths ------------------------------------------------------
    def all_gather_into(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        if self._host_staged and out.is_cuda:
            h = torch.empty(out.shape, dtype=out.dtype)
            dist.all_gather_into_tensor(h, inp.cpu(), group=self.group)
            out.copy_(h)
            return
        dist.all_gather_into_tensor(out, inp, group=self.group)

    def all_to_all_into(self, out: torch.Tensor, inp: torch.Tensor, async_op: bool = False):
        if self._host_staged and out.is_cuda:
            h = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(h, inp.cpu(), group=self.group)
            out.copy_(h)
            return _DoneWork()
        work = dist.all_to_all_single(out, inp, group=self.group, async_op=async_op)
        return work if async_op else _DoneWork()

    # -- reference-compatible API -----------------------------------------
    def all_gather(self, local: torch.Tensor) -> torch.Tensor:
        if local.dim() != 2:
            raise CollectiveContractError(f"all_gather expects a 2-D matrix, got ndim={local.dim()}")
        local = local.contiguous()
        out = torch.empty((self.world_size * local.shape[0], *local.shape[1:]),
                          dtype=local.dtype, device=local.device)
        self.all_gather_into(out, local)
        return out

    def all_reduce(self, buffer: torch.Tensor, op=ReduceOp.SUM) -> torch.Tensor:
        op = _as_op(op)
        buffer = buffer.contiguous()
        flat = buffer.reshape(1, -1)
        gathered = self.all_gather(flat)
        return _ordered_reduce(list(gathered.unbind(0)), op).reshape(buffer.shape)

    def all_reduce_scalar(self, value: float, op=ReduceOp.SUM) -> float:
        op = _as_op(op)
        dev = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        t = torch.tensor([[float(value)]], dtype=torch.float64, device=dev)
        vals = self.all_gather(t).reshape(-1).tolist()
        acc = float(vals[0])
        for v in vals[1:]:
            acc += v
        if op is ReduceOp.AVG:
            acc /= self.world_size
        return acc

    def barrier(self) -> None:
        dist.barrier(group=self.group)


# ---------------------------------------------------------------------------
# Simulated ranks on one device (threads)
# ---------------------------------------------------------------------------
class _Round:
    def __init__(self, world_size: int, kind: str, sig):
        self.kind = kind
        self.sig = sig
        self.slots = [None] * world_size
        self.arrived = set()
        self.done = False
        self.result = None


class LocalGroup:
    """Rendezvous for ``world_size`` rank threads sharing one CUDA device."""

    def __init__(self, world_size: int, timeout: float = DEFAULT_TIMEOUT, peer: bool = False):
        if world_size < 1:
            raise ValueError(f"world size must be >= 1, got {world_size}")
        self.world_size = world_size
        self.peer = peer
        self.timeout = timeout
        self._cond = threading.Condition()
        self._round = None
        self._error = None

    def endpoint(self, rank: int) -> "LocalEndpoint":
        if not 0 <= rank < self.world_size:
            raise ValueError(f"rank {rank} outside [0, {self.world_size})")
        return LocalEndpoint(self, rank)

    def poison(self, error: BaseException) -> None:
        with self._cond:
            if self._error is None:
                self._error = error
            self._cond.notify_all()

    def collective(self, rank: int, kind: str, payload, sig, finalize):
        with self._cond:
            if self._error is not None:
                raise self._error
            rnd = self._round
            if rnd is None:
                rnd = self._round = _Round(self.world_size, kind, sig)
            elif rnd.kind != kind or rnd.sig != sig:
                err = CollectiveContractError(
                    f"rank {rank} entered {kind} {sig} while the group is in {rnd.kind} {rnd.sig}")
                self._error = err
                self._cond.notify_all()
                raise err
            rnd.slots[rank] = payload
            rnd.arrived.add(rank)
            if len(rnd.arrived) == self.world_size:
                rnd.result = finalize(rnd.slots)
                rnd.done = True
                self._round = None
                self._cond.notify_all()
            else:
                deadline = time.monotonic() + self.timeout
                while not rnd.done and self._error is None:
                    remaining = deadline - time.monotonic()
                    if remaining <= 0:
                        missing = tuple(sorted(set(range(self.world_size)) - rnd.arrived))
                        err = CollectiveTimeoutError(
                            f"{kind} timed out after {self.timeout:g}s; missing ranks {list(missing)}",
                            missing)
                        self._error = err
                        self._cond.notify_all()
                        raise err
                    self._cond.wait(remaining)
                if self._error is not None:
                    raise self._error
            return rnd.result


def _record(t: torch.Tensor):
    if t.is_cuda:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(t.device))
        return ev
    return None


def _wait_all(events, device):
    if device.type == "cuda":
        s = torch.cuda.current_stream(device)
        for ev in events:
            if ev is not None:
                s.wait_event(ev)


def _done_event(device):
    if device.type == "cuda":
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(device))
        return ev
    return None


class LocalEndpoint:
    """One simulated rank; owned by exactly one thread."""

    in_process = True  # peer windows are shared as raw device pointers

    def __init__(self, group: LocalGroup, rank: int):
        self.group = group
        self.rank = rank
        self.peer = group.peer

    def exchange(self, obj) -> list:
        """All ranks' objects, in rank order."""
        return self.group.collective(self.rank, "exchange", obj, (), lambda slots: list(slots))

    @property
    def world_size(self) -> int:
        return self.group.world_size

    def _finish(self, done):
        if done is not None:
            torch.cuda.current_stream().wait_event(done)

    def all_gather_into(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        payload = (out, inp, _record(inp))

        def finalize(slots):
            dev = slots[0][1].device
            _wait_all([s[2] for s in slots], dev)
            n = slots[0][1].numel()
            for o, _, _ in slots:
                flat = o.view(-1)
                for r, (_, i, _) in enumerate(slots):
                    flat[r * n:(r + 1) * n].copy_(i.reshape(-1))
            return _done_event(dev)

        self._finish(self.group.collective(self.rank, "all_gather_into", payload,
                                           (inp.numel(), inp.dtype), finalize))

    def all_to_all_into(self, out: torch.Tensor, inp: torch.Tensor, async_op: bool = False):
        payload = (out, inp, _record(inp))
        world = self.world_size

        def finalize(slots):
            dev = slots[0][1].device
            _wait_all([s[2] for s in slots], dev)
            n = slots[0][1].numel() // world
            for dst, (o, _, _) in enumerate(slots):
                of = o.view(-1)
                for src, (_, i, _) in enumerate(slots):
                    of[src * n:(src + 1) * n].copy_(i.reshape(-1)[dst * n:(dst + 1) * n])
            return _done_event(dev)

        self._finish(self.group.collective(self.rank, "all_to_all_into", payload,
                                           (inp.numel(), inp.dtype), finalize))
        return _DoneWork()

    def all_gather(self, local: torch.Tensor) -> torch.Tensor:
        if local.dim() != 2:
            raise CollectiveContractError(f"all_gather expects a 2-D matrix, got ndim={local.dim()}")
        local = local.contiguous()
        out = torch.empty((self.world_size * local.shape[0], *local.shape[1:]),
                          dtype=local.dtype, device=local.device)
        self.all_gather_into(out, local)
        return out

    def all_reduce(self, buffer: torch.Tensor, op=ReduceOp.SUM) -> torch.Tensor:
        op = _as_op(op)
        payload = (buffer.contiguous(), _record(buffer))

        def finalize(slots):
            dev = slots[0][0].device
            _wait_all([s[1] for s in slots], dev)
            res = _ordered_reduce([s[0] for s in slots], op)
            return res, _done_event(dev)

        res, done = self.group.collective(self.rank, "all_reduce", payload,
                                          (tuple(buffer.shape), buffer.dtype, op), finalize)
        self._finish(done)
        return res

    def all_reduce_scalar(self, value: float, op=ReduceOp.SUM) -> float:
        op = _as_op(op)

        def finalize(slots):
            acc = float(slots[0])
            for v in slots[1:]:
                acc += v
            if op is ReduceOp.AVG:
                acc /= len(slots)
            return acc

        return self.group.collective(self.rank, "all_reduce_scalar", float(value), (op,), finalize)

    def barrier(self) -> None:
        self.group.collective(self.rank, "barrier", None, (), lambda slots: None)


class SingleEndpoint:
    """World size 1: every collective is the identity."""

    rank = 0
    world_size = 1

    def all_gather_into(self, out, inp):
        out.view(-1).copy_(inp.reshape(-1))

    def all_to_all_into(self, out, inp, async_op=False):
        out.view(-1).copy_(inp.reshape(-1))
        return _DoneWork()

    def all_gather(self, local):
        return local

    def all_reduce(self, buffer, op=ReduceOp.SUM):
        return buffer

    def all_reduce_scalar(self, value, op=ReduceOp.SUM):
        return float(value)

    def barrier(self):
        return None


def run_ranks(world_size: int, fn, *, device=None, timeout: float = DEFAULT_TIMEOUT, peer: bool = False,
              own_streams: bool = False) -> list:
    """Run ``fn(endpoint)`` once per simulated rank (threads, one device); return results.

    Same contract as the reference's run_ranks (fabric.py:291-324): the first
    failing rank's exception is re-raised after all workers stop.  ``peer=True`` routes the
    gradient exchange through the peer transport (windows shared as device pointers); each rank
    thread then runs on its own CUDA stream.
    """
    group = LocalGroup(world_size, timeout=timeout, peer=peer)
    own_streams = own_streams or peer  # the peer transport's wait kernels need independent rank streams
    results = [None] * world_size
    errors = [None] * world_size
    dev = device if device is not None else (torch.cuda.current_device() if torch.cuda.is_available() else None)

    def worker(rank: int) -> None:
        try:
            if dev is not None:
                torch.cuda.set_device(dev)
            if own_streams:  # ranks progress independently (the peer transport waits on device flags)
                with torch.cuda.stream(torch.cuda.Stream()):
                    results[rank] = fn(group.endpoint(rank))
                    torch.cuda.current_stream().synchronize()
            else:
                results[rank] = fn(group.endpoint(rank))
        except BaseException as exc:  # propagate to the caller, unblock peers
            errors[rank] = exc
            group.poison(exc)

    threads = [threading.Thread(target=worker, args=(r,), name=f"rank-{r}", daemon=True)
               for r in range(world_size)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for exc in errors:
        if exc is not None:
            raise exc
    return results
