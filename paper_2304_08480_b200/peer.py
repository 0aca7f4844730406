"""Peer transport: the cross-rank gradient exchange over NVLink peer memory.

Replaces the reference's all_reduce(AVG) of the two B x D contributions + row slice
(shard.py:199-208) -- realised on the default path as an NCCL all_to_all of fp32 slabs plus a
fixed-order tree -- by pushes from inside the backward GEMM: each cross tile's epilogue
TMA-stores its chunk partial straight into the owning rank's peer window, a one-warp kernel
publishes an arrival epoch to every owner, and the owner's combine waits for all N epochs and
sums the leaves in the same fixed tree (include/disco_b200.h, "Peer transport").  The result is
bit-identical to the all_to_all path and to N = 1.

Windows are one cudaMalloc per rank (disco_b200_peer_alloc).  Across processes the bases are
shared as CUDA IPC handles through the endpoint's object exchange; simulated ranks (threads of
one process, ``LocalGroup(peer=True)``) share raw device pointers.
"""

import ctypes
import os

from . import _lib

# wait-kernel bound: a missing peer sets status flag 8 (CollectiveTimeoutError) instead of a hang
PEER_TIMEOUT_S = float(os.environ.get("DISCO_PEER_TIMEOUT", "60"))


def enabled(endpoint) -> bool:
    """Peer transport on for this endpoint: ``endpoint.peer`` if set, else env DISCO_PEER
    (default on; DISCO_PEER=0 selects the NCCL all_to_all + sender presum exchange)."""
    flag = getattr(endpoint, "peer", None)
    if flag is None:
        flag = os.environ.get("DISCO_PEER", "1") not in ("", "0")
    return bool(flag) and endpoint.world_size > 1


def streamed_gather(endpoint, B: int, world: int) -> bool:
    """The all-gather overlapped with the logits GEMM (copy-engine pulls + flag-gated persistent
    kernel).  Opt-in (DISCO_PEER_STREAMED=1) and one process per GPU only: when ranks share a GPU
    (threads of one process, or the two-process single-GPU check) one rank's spinning kernel can
    hold the SMs the other rank's publish needs -- measured to time out at B=8192 on one GPU; with
    a GPU per rank that cannot happen, but the path is not yet validated on NVLink."""
    if getattr(endpoint, "in_process", False) or os.environ.get("DISCO_PEER_STREAMED", "0") in ("", "0"):
        return False
    return B % 1024 == 0 and 8 % world == 0  # canonical chunks


def supported(B: int, D: int, world: int, rank: int) -> bool:
    if world < 2 or world > 8 or B % world or (B // world) % 128:
        return False
    return True


def in_process_fence(endpoint, stream) -> None:
    """Simulated ranks (threads sharing ONE GPU, ``endpoint.in_process``): order every rank's
    signalled work before any rank's wait kernel, so a wait kernel never spins.

    On one shared device a spinning wait kernel can deadlock against a peer thread's allocation:
    a device/pinned-memory allocation implicitly serialises the streams, so a publish enqueued
    after another thread's ``cudaMalloc`` waits for the spinning kernel that waits for it (seen as
    a 60 s wait timeout with garbage operands on a CPU-contended box).  Each rank records an event
    after its signal, the events are exchanged through the host rendezvous and every rank's stream
    waits on all of them: the wait kernels still read the device flags (the protocol is unchanged)
    but find them already raised.  Processes with a GPU each never take this path."""
    if not getattr(endpoint, "in_process", False):
        return
    import torch
    ev = torch.cuda.Event()
    ev.record(stream)
    for e in endpoint.exchange(ev):
        stream.wait_event(e)


def window_bytes(B: int, D: int, world: int, rank: int) -> int:
    """Size of a rank's peer window for the geometry (and backward mode) the library sees now."""
    n = ctypes.c_int64()
    _lib.call("disco_b200_peer_bytes", B, D, world, rank, ctypes.byref(n))
    return n.value


class PeerUnavailable(RuntimeError):
    """The peer transport cannot run on this group (no peer access between some pair of GPUs, or
    the IPC mapping failed on some rank).  Raised on EVERY rank (the decision is collective), so
    the caller can fall back to the NCCL exchange without a rank hanging in a wait kernel."""


def _peer_access_all_pairs(devices) -> bool:
    import torch
    for i in set(devices):
        for j in set(devices):
            if i != j and not torch.cuda.can_device_access_peer(i, j):
                return False
    return True


class PeerWindow:
    """This rank's peer window and the N window bases (index = rank) for one plan geometry."""

    def __init__(self, endpoint, B: int, D: int, world: int, rank: int):
        import torch
        lib = _lib.load()
        self.world, self.rank = world, rank
        self.base = None
        self._opened = []
        in_process = getattr(endpoint, "in_process", False)
        if not in_process:
            # every rank sees every rank's device: identical all-pairs answer on every rank
            devices = endpoint.exchange(torch.cuda.current_device())
            if not _peer_access_all_pairs(devices):
                raise PeerUnavailable(f"no peer access between some pair of GPUs {sorted(set(devices))}")
        self.nbytes = window_bytes(B, D, world, rank)
        handle = None if in_process else ctypes.create_string_buffer(lib.disco_b200_peer_handle_bytes())
        ptr = ctypes.c_void_p()
        _lib.call("disco_b200_peer_alloc", self.nbytes, ctypes.byref(ptr), handle)
        self.base = ptr.value
        try:
            if in_process:
                bases = endpoint.exchange(self.base)
            else:
                handles = endpoint.exchange(bytes(handle.raw))
                bases, err = [], None
                for r, h in enumerate(handles):
                    if r == rank:
                        bases.append(self.base)
                        continue
                    p = ctypes.c_void_p()
                    try:
                        _lib.call("disco_b200_peer_open", ctypes.create_string_buffer(h, len(h)), ctypes.byref(p))
                    except RuntimeError as exc:
                        err = str(exc)
                        break
                    self._opened.append(p.value)
                    bases.append(p.value)
                failures = [e for e in endpoint.exchange(err) if e]  # collective: all ranks decide alike
                if failures:
                    raise PeerUnavailable(f"peer window mapping failed: {failures[0]}")
        except BaseException:
            self.close()
            raise
        self.bases = (ctypes.c_uint64 * world)(*bases)
        self.epoch = 0
        endpoint.barrier()  # every window's arrival flags are zeroed before any rank signals

    def next_step(self):
        """(epoch, parity) of the next step; every rank advances in lockstep."""
        self.epoch = (self.epoch + 1) & 0xFFFFFFFF or 1
        return self.epoch, self.epoch & 1

    def close(self) -> None:
        lib = _lib.load()
        for p in self._opened:
            lib.disco_b200_peer_close(ctypes.c_void_p(p))
        self._opened = []
        if self.base:
            lib.disco_b200_peer_free(ctypes.c_void_p(self.base))
            self.base = None
