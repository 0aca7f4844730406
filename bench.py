#!/usr/bin/env python3
"""Benchmark: DisCo contrastive-loss fwd+bwd samples/sec at B=32K, D=512 (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1; one rank per GPU, NCCL)

A step is one DisCo loss forward+backward over the global batch (B=32768
image/text pairs, D=512, t=100): every rank runs disco_step on its b = B/N
rows (shard.py:169-208).  Workload = BASELINE.json configs[1] (strong
scaling: B fixed, N varies).

Printed on rank 0, one JSON line:
  value     samples/s = B / t_step, t_step = max over ranks of the device time
            of the step (inputs resident in HBM, CUDA events per step, L2
            flushed between steps outside the timed events).
  e2e       same metric through the public API with HOST (pinned, bf16)
            inputs and host outputs: H2D of the features, D2H of both fp32
            gradient blocks and the loss inside the timed region.
  roofline  dominant kernel: algorithmic FLOPs per launch / mean launch time
            (CUDA events on the launching stream) against the measured bf16
            peak (MEASURED_PEAKS.json); step-level fraction alongside.
  cpu_baseline  the oracle port of the reference path (oracle/disco_oracle.py,
            numpy f32, all host cores), one full step (rank 0, N=1 only).
  exchange_backward  (N=1) the same step with DISCO_BACKWARD=exchange: intra + cross
            GEMMs, the reference's dataflow; `value` is the default dual backward.
``--impl reference`` times that CPU port (full steps) as the reference arm, plus one
step of the unmodified reference disco_step from baseline/_ref when installed.
"""

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B_GLOBAL = 32768
DIM = 512
TEMP = 100.0
# BASELINE.json configs (B, D): 1 = headline; 2-4 are extra measurement points
CONFIGS = {"A": (1024, 512), "B": (32768, 512), "C": (65536, 768), "D": (196608, 512), "E": (16384, 1024)}
METRIC = "contrastive-loss fwd+bwd samples/sec at B=32K,D=512; peak loss mem/GPU"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--dim", type=int, default=None)
    ap.add_argument("--config", default="B", choices=sorted(CONFIGS),
                    help="BASELINE.json config letter (SURVEY 8.0); --batch/--dim override")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-exchange-leg", "--no-fused", dest="no_exchange_leg", action="store_true",
                    help="skip the exchange-backward comparison leg (N = 1)")
    ap.add_argument("--no-ref-check", action="store_true",
                    help="reference arm: skip the one-step cross-check of the other CPU implementation")
    ap.add_argument("--cpu-port", action="store_true",
                    help="time the oracle port even when the unmodified reference (baseline/_ref) is installed")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm on the host cores, FULL workload per step
# ---------------------------------------------------------------------------
def cpu_features(B, D, seed=0):
    """cli.py:103-105 features, bf16-rounded, as f32 (the reference's benchmark precision,
    costs.py:158)."""
    from oracle import disco_oracle as O
    rng = np.random.default_rng(seed)
    I = rng.standard_normal((B, D)).astype(np.float32)
    I /= np.linalg.norm(I, axis=1, keepdims=True)
    T = rng.standard_normal((B, D)).astype(np.float32)
    T /= np.linalg.norm(T, axis=1, keepdims=True)
    return O.bf16_round(I), O.bf16_round(T)


def cpu_port_step(I, T, world, t=TEMP, workers=None):
    """One full DisCo step of all `world` ranks on the host (oracle.disco_step_blocked: the
    reference's shard.py:98-208 arithmetic in f32, row blocks on `workers` threads with
    single-threaded BLAS each).  Returns seconds."""
    from oracle import disco_oracle as O
    from threadpoolctl import threadpool_limits
    workers = workers or cpu_cores()
    t0 = time.perf_counter()
    with threadpool_limits(1):
        d_i, d_t, loss = O.disco_step_blocked(I, T, world, t, rows_per_block=512, workers=workers)
    sec = time.perf_counter() - t0
    assert np.isfinite(loss)
    return sec


def _reference_package():
    """The UNMODIFIED reference package installed in baseline/_ref (python -m pip install --no-index
    --no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>), or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "disco")):
        return None
    sys.path.insert(0, ref)
    try:
        import disco  # the reference package, unmodified
        from disco import disco_step, run_ranks  # noqa: F401
    except Exception:
        return None
    finally:
        sys.path.remove(ref)
    return disco


def unmodified_reference_step(I, T, world, t=TEMP):
    """One step of the UNMODIFIED reference disco_step (shard.py:169-208) for all `world` ranks
    through its own run_ranks (fabric.py:291, lockstep) with verification on, f32 features, all
    host cores (numpy / OpenBLAS as shipped).  Returns seconds, or None without baseline/_ref."""
    disco = _reference_package()
    if disco is None:
        return None
    b = I.shape[0] // world

    def fn(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        return disco.disco_step(ep, I[rows], T[rows], t)[2]

    t0 = time.perf_counter()
    disco.run_ranks(world, fn, mode="lockstep")
    return time.perf_counter() - t0


def reference_kind(args) -> str:
    """'reference' (the unmodified package from baseline/_ref) when installed, else 'port'."""
    if getattr(args, "cpu_port", False) or _reference_package() is None:
        return "port"
    return "reference"


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    """The reference arm: the reference's own CPU implementation of the step on the host cores --
    the unmodified package from baseline/_ref (kind "reference") when installed, else the
    vectorised oracle port (kind "port") -- every one of the W + K steps the FULL workload (all
    B rows, both directions); the other implementation is timed once beside it as a cross-check."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    B, D, N = args.batch, args.dim, args.gpus
    I, T = cpu_features(B, D)
    cores = cpu_cores()
    kind = reference_kind(args)
    step = unmodified_reference_step if kind == "reference" else cpu_port_step
    t_start = time.perf_counter()
    for _ in range(args.warmup):
        step(I, T, N)
    secs = [step(I, T, N) for _ in range(args.steps)]
    wall = time.perf_counter() - t_start
    sec = statistics.mean(secs)
    value = B / sec
    cross = None
    if not args.no_ref_check:
        if kind == "reference":
            ps = cpu_port_step(I, T, N)
            cross = {"kind": "port", "value": B / ps, "unit": UNIT, "ms_per_step": 1e3 * ps, "steps": 1,
                     "note": "oracle.disco_step_blocked (f32, row blocks on all host threads, no verification pass)"}
        else:
            us = unmodified_reference_step(I, T, N)
            if us is not None:
                cross = {"kind": "reference", "value": B / us, "unit": UNIT, "ms_per_step": 1e3 * us, "steps": 1}
    if kind == "reference":
        sample = (f"full step: unmodified reference disco_step (shard.py:169-208) for all {N} rank(s) via "
                  f"run_ranks(lockstep), verification on, {B // N} rows x {B} columns, D={D}, f32, "
                  f"numpy/OpenBLAS on {cores} cores")
    else:
        sample = (f"full step: all {N} rank(s) x {B // N} rows x {B} columns, D={D}, both directions "
                  f"(oracle.disco_step_blocked, f32, {cores} threads x 1-thread BLAS)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(args, B, D, N),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                         "cross_check": cross},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, B, D, world):
    """The `config` object both arms print (same keys, so the driver can pair the lines)."""
    return {"workload": f"B={B},D={D},t={TEMP} (BASELINE config {args.config})", "global_batch": B,
            "local_batch": B // world, "dim": D, "parallelism": f"dp{world}"}


# ---------------------------------------------------------------------------
# clocks sampler (NVML) during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as exc:  # pragma: no cover
            self.err = str(exc)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.01)

    def __enter__(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.th.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["bf16_tflops"], pk.get("bf16_tflops_sustained", pk["bf16_tflops"]), pk["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def load_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


def exchange_preflight(P, ep, I, T, t, world, local_rank, share):
    """Decide the N > 1 exchange before the timed steps (never fatal).

    The peer transport (default) needs peer access between every pair of GPUs and working CUDA
    IPC windows.  Check ``can_device_access_peer`` for all pairs, then run one step through the
    NCCL exchange (DISCO_PEER=0 path) and one through the peer transport and require identical
    bytes (both are bitwise equal to N = 1 by construction).  Any failure, timeout or mismatch
    on any rank selects the NCCL exchange for the whole job; the choice and the reason are
    recorded in ``config.exchange_preflight``."""
    import torch
    import torch.distributed as dist
    from paper_2304_08480_b200 import peer as peer_mod
    from paper_2304_08480_b200.shard import clear_plans

    B, D = I.shape[0] * world, I.shape[1]
    info = {"peer_requested": peer_mod.enabled(ep), "peer_supported": peer_mod.supported(B, D, world, ep.rank)}
    dev = torch.device("cuda", local_rank)

    def agree(ok: bool) -> bool:  # every rank must agree (MIN over ranks)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev if not share else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        return bool(flag.item())

    if share:
        access = True  # every rank on cuda:0 (code-path check)
    else:
        n_dev = torch.cuda.device_count()
        access = all(torch.cuda.can_device_access_peer(local_rank, j) for j in range(min(world, n_dev)) if j != local_rank)
    info["peer_access_all_pairs"] = agree(access)
    if not (info["peer_requested"] and info["peer_supported"]):
        info.update(choice="nccl", reason="peer transport not requested or not supported for this geometry")
        ep.peer = False
        return info
    if not info["peer_access_all_pairs"]:
        info.update(choice="nccl", reason="cudaDeviceCanAccessPeer false for some GPU pair")
        ep.peer = False
        return info
    ref, err = None, None
    try:
        ep.peer = False
        di0, dt0, l0 = P.disco_step(ep, I, T, t)
        ref = (di0.clone(), dt0.clone(), l0)
    except Exception as exc:  # pragma: no cover - reported, then the job decides below
        err = f"nccl step failed: {type(exc).__name__}: {exc}"
    same = False
    saved_timeout = peer_mod.PEER_TIMEOUT_S
    if ref is not None:
        peer_mod.PEER_TIMEOUT_S = 20.0  # a broken transport raises CollectiveTimeoutError, never hangs
        try:
            ep.peer = True
            for _ in range(2):  # both parity windows
                di1, dt1, l1 = P.disco_step(ep, I, T, t)
            same = bool(torch.equal(di1, ref[0]) and torch.equal(dt1, ref[1]) and l1 == ref[2])
            if not same:
                err = "peer step differs from the NCCL step"
        except Exception as exc:
            err = f"peer step failed: {type(exc).__name__}: {exc}"
        finally:
            peer_mod.PEER_TIMEOUT_S = saved_timeout
    try:
        ok = agree(same)
    except Exception as exc:  # pragma: no cover
        ok, err = False, f"agreement collective failed: {exc}"
    info["peer_step_matches_nccl"] = ok
    ep.peer = ok
    if not ok:
        clear_plans()
    info.update(choice="peer" if ok else "nccl", reason=err if not ok else "peer access + bitwise-equal preflight step")
    return info


def phase_breakdown(P, _lib, peer_mod, ep, plan, names, I, T, t, st, flush, barrier, use_peer, dual, reps=5):
    """Mean ms of each C-ABI phase of one step (CUDA events around each call on the launch stream,
    L2 flushed before every rep); `names` selects the phases of the path being measured."""
    import torch
    B, D, world = plan.B, plan.D, plan.world
    b = B // world
    args_ = plan.args
    sp = st.cuda_stream
    dev = plan.device
    ev = {n: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for n in names}
    acc = {n: 0.0 for n in names}
    di = torch.empty((b, D), dtype=torch.float32, device=dev)
    dt_ = torch.empty((b, D), dtype=torch.float32, device=dev)

    def timed(name, fn):
        if name not in ev:
            return
        ev[name][0].record(st)
        fn()
        ev[name][1].record(st)

    for _ in range(reps):
        flush.zero_()
        barrier()
        timed("pack", lambda: _lib.call("disco_b200_pack", *args_, I.data_ptr(), T.data_ptr(), D, D, _lib.BF16, 1, sp))
        timed("all_gather", lambda: ep.all_gather_into(plan.gather, plan.pack))
        pw = parity = epoch = None
        if use_peer:
            pw = plan.peer_window(ep)
            epoch, parity = pw.next_step()
            timed("peer_gather", lambda: (_lib.call("disco_b200_peer_publish", *args_, pw.bases, parity, epoch, sp),
                                          _lib.call("disco_b200_peer_gather", *args_, pw.bases, parity, epoch,
                                                    peer_mod.PEER_TIMEOUT_S, sp)))
            timed("forward", lambda: _lib.call("disco_b200_forward_gathered", *args_, t, sp))
        else:
            timed("forward", lambda: _lib.call("disco_b200_forward", *args_, t, sp))
        if dual:
            timed("stats_exchange", lambda: ep.all_gather_into(plan.xall, plan.xchg))
            timed("dual_prep", lambda: _lib.call("disco_b200_dual_prep", *args_, 0, sp))
            timed("backward", lambda: _lib.call("disco_b200_backward_dual", *args_, 0, b, sp))
            timed("combine", lambda: _lib.call("disco_b200_combine_dual", *args_, t, 0, b, di.data_ptr(),
                                               dt_.data_ptr(), D, sp))
            timed("fixup", lambda: _lib.call("disco_b200_dual_fixup", *args_, t, 0, di.data_ptr(), dt_.data_ptr(),
                                             D, sp))
            timed("loss", lambda: _lib.call("disco_b200_loss", *args_, 2, sp))
        else:
            timed("backward_grad", lambda: _lib.call("disco_b200_backward_grad", *args_, t, sp))
            timed("backward", lambda: _lib.call("disco_b200_backward_fused", *args_, sp))
            if use_peer:
                timed("backward_peer", lambda: _lib.call("disco_b200_backward_peer", *args_, pw.bases, parity, epoch,
                                                         sp))
                timed("combine_peer", lambda: _lib.call("disco_b200_combine_peer", *args_, t, 0, pw.base, parity,
                                                        epoch, peer_mod.PEER_TIMEOUT_S, di.data_ptr(), dt_.data_ptr(),
                                                        D, sp))
            timed("backward_cross", lambda: _lib.call("disco_b200_backward_cross", *args_, sp))
            timed("all_to_all", lambda: ep.all_to_all_into(plan.recv, plan.send))
            timed("backward_intra", lambda: _lib.call("disco_b200_backward_intra", *args_, sp))
            timed("combine", lambda: _lib.call("disco_b200_combine", *args_, t, 0, di.data_ptr(), dt_.data_ptr(), D,
                                               sp))
            if use_peer:  # the ce rode with the slabs into this rank's window
                timed("loss", lambda: _lib.call("disco_b200_loss_peer", *args_, pw.base, parity, sp))
            else:
                timed("loss", lambda: (world > 1 and ep.all_gather_into(plan.ce_all, plan.ce),
                                       _lib.call("disco_b200_loss", *args_, 0, sp)))
        torch.cuda.synchronize()
        for n in names:
            acc[n] += ev[n][0].elapsed_time(ev[n][1]) / reps
    return {n: round(v, 4) for n, v in acc.items()}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # DISCO_BENCH_SHARE_GPU=1 (code-path check only, numbers meaningless): every rank on cuda:0,
    # gloo for the host plumbing -- exercises the N > 1 bench path on a one-GPU box
    share = os.environ.get("DISCO_BENCH_SHARE_GPU", "0") == "1"
    if share:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)

    import paper_2304_08480_b200 as P
    from paper_2304_08480_b200 import _lib
    from paper_2304_08480_b200.shard import get_plan

    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)
        ep = P.ProcessGroupEndpoint()
    else:
        ep = P.SingleEndpoint()

    B, D, t = args.batch, args.dim, TEMP
    b = B // world
    # synthetic features (cli.py:103-105 distribution), bf16, this rank's rows only
    g = torch.Generator(device=device)
    g.manual_seed(1234 + rank)
    I = torch.randn(b, D, device=device, generator=g)
    T = torch.randn(b, D, device=device, generator=g)
    I = (I / I.norm(dim=1, keepdim=True)).to(torch.bfloat16)
    T = (T / T.norm(dim=1, keepdim=True)).to(torch.bfloat16)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=device)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- N > 1: check the peer transport before trusting it with the timed steps -------------
    preflight = exchange_preflight(P, ep, I, T, TEMP, world, local_rank, share) if world > 1 else None
    from paper_2304_08480_b200.shard import clear_plans
    clear_plans()
    torch.cuda.empty_cache()

    # ---- loss-scope memory: everything the first step allocates (workspace incl. the O(B^2/N)
    # E/G blocks, outputs), measured by the caching allocator from a clean slate -----------
    torch.cuda.synchronize()
    mem_before = torch.cuda.memory_allocated(device)
    torch.cuda.reset_peak_memory_stats(device)
    plan = get_plan(B, D, world, rank, device)
    st = torch.cuda.current_stream(device)

    def step():
        return P.disco_step_async(ep, I, T, t)

    step()
    P.finish_status(plan)
    torch.cuda.synchronize()
    loss_mem = torch.cuda.max_memory_allocated(device) - mem_before
    g_off, g_bytes_ws = _lib.ws_region(B, D, world, rank, _lib.R_G)
    for _ in range(args.warmup):
        step()
    P.finish_status(plan)
    torch.cuda.synchronize()

    # ---- timed region: K steps, each bracketed by CUDA events -------------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush outside the timed events
            starts[i].record(st)
            step()
            ends[i].record(st)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    barrier()
    loss = P.finish_status(plan)
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = statistics.mean(step_ms)
    peak_mem = torch.cuda.max_memory_allocated(device)
    if world > 1:
        tt = torch.tensor([ms], device=device, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = B / (ms / 1e3)

    # ---- kernel breakdown: events around each C-ABI call (one tensor-core kernel each)
    from paper_2304_08480_b200 import peer as peer_mod
    use_peer = world > 1 and peer_mod.enabled(ep) and peer_mod.supported(B, D, world, rank)
    dual = bool(_lib.path_info(B, D, world, rank) & _lib.PATH_DUAL)
    names = ["pack"] + (["peer_gather"] if use_peer else ["all_gather"] if world > 1 else []) + ["forward"]
    if dual:  # the default: statistics exchange, one GEMM per gradient over the rank's own E block
        names += (["stats_exchange"] if world > 1 else []) + ["dual_prep", "backward", "combine", "fixup", "loss"]
    elif world == 1:  # exchange backward, intra + cross as one launch
        names += ["backward_grad", "backward", "combine", "loss"]
    elif use_peer:  # fused intra + cross GEMM pushing cross tiles to the owners
        names += ["backward_grad", "backward_peer", "combine_peer", "loss"]
    else:
        names += ["backward_grad", "backward_cross", "all_to_all", "backward_intra", "combine", "loss"]
    phases = phase_breakdown(P, _lib, peer_mod, ep, plan, names, I, T, t, st, flush, barrier, use_peer, dual)
    traffic_n = None
    peer_bytes = 0
    if world > 1:
        from paper_2304_08480_b200 import costs as costs_mod
        Dp = (D + 63) // 64 * 64
        ag_bytes = (world - 1) * 2 * b * Dp * 2   # bf16 rows received per rank (both feature sets)
        link = 900.0                              # NVLink 5 GB/s per direction
        ag_ms = phases.get("peer_gather", phases.get("all_gather"))
        traffic_n = {"note": "bytes per rank per step; busbw = bytes moved per rank / phase time "
                             "(nccl-tests convention: algbw * (N-1)/N); link = 900 GB/s per direction",
                     "all_gather": {"bytes": ag_bytes, "ms": ag_ms, "busbw_gbs": ag_bytes / (ag_ms / 1e3) / 1e9,
                                    "frac_of_link": ag_bytes / (ag_ms / 1e3) / 1e9 / link,
                                    "kind": "peer pull + unpack kernel" if use_peer else "nccl all_gather_into_tensor"}}
        if dual:
            sx_bytes = (world - 1) * 4 * b * 4
            traffic_n["stats_exchange"] = {
                "bytes": sx_bytes, "ms": phases["stats_exchange"],
                "kind": "nccl all_gather of the 4 b per-row statistics (lse2, ce); the dual backward "
                        "needs no gradient reduce-scatter"}
        elif use_peer:
            rs_bytes = (world - 1) * 2 * b * Dp * 4   # fp32 partial rows each rank sends to their owners
            bw_ms = phases["backward_peer"]
            traffic_n["reduce_scatter"] = {
                "bytes": rs_bytes, "ms_overlapped": bw_ms, "combine_ms": phases["combine_peer"],
                "push_gbs_during_gemm": rs_bytes / (bw_ms / 1e3) / 1e9,
                "kind": "TMA pushes from the backward GEMM epilogue into the owners' windows (overlapped)"}
        else:
            rs_bytes = (world - 1) * 2 * b * Dp * 4
            a_ms = phases["all_to_all"]
            traffic_n["reduce_scatter"] = {"bytes": rs_bytes, "ms": a_ms, "busbw_gbs": rs_bytes / (a_ms / 1e3) / 1e9,
                                           "frac_of_link": rs_bytes / (a_ms / 1e3) / 1e9 / link,
                                           "kind": "nccl all_to_all_single of fp32 destination slabs"}
        if use_peer:
            peer_bytes = costs_mod.peer_window_bytes(B, D, world, rank)
    kernel_mhz = _lib.clock_probe(plan)  # SM clock the last timed launches actually ran at

    # ---- e2e through the public API with host buffers ---------------------
    def measure_e2e():
        I_h = I.cpu().pin_memory()
        T_h = T.cpu().pin_memory()
        for _ in range(2):
            P.disco_step(ep, I_h, T_h, t)
        e_ms = []
        barrier()
        for _ in range(max(3, args.steps // 2)):
            flush.zero_()
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(st)
            di_h, dt_h, _ = P.disco_step(ep, I_h, T_h, t)
            s1.record(st)
            s1.synchronize()
            e_ms.append(s0.elapsed_time(s1))
            out_bytes = int(di_h.numel() * 4 * 2 + 8)
            del di_h, dt_h  # the caller consumes and drops the host gradients each step
        em = statistics.mean(e_ms)
        if world > 1:
            tt = torch.tensor([em], device=device, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            em = float(tt.item())
        return {"value": B / (em / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(I_h.numel() * I_h.element_size() * 2),
                "d2h_bytes_per_step": out_bytes,
                "ms_per_step": em}

    e2e = None if args.no_e2e else measure_e2e()

    # ---- the exchange backward (DISCO_BACKWARD=exchange), same workload, for comparison -----
    # Intra + cross GEMMs (8*b*B*D backward flops) and, at N > 1, the gradient reduce-scatter: the
    # reference's dataflow (shard.py:148-154, 199-208).  The line's `value` is the dual backward.
    exchange = None
    if world == 1 and dual and not args.no_exchange_leg:
        saved = os.environ.get("DISCO_BACKWARD")
        os.environ["DISCO_BACKWARD"] = "exchange"
        try:
            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize()
            f0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            f1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            for i in range(args.steps):
                flush.zero_()
                f0[i].record(st)
                step()
                f1[i].record(st)
            torch.cuda.synchronize()
            fms = statistics.mean(a.elapsed_time(z) for a, z in zip(f0, f1))
            x_loss = P.finish_status(plan)
            xph = phase_breakdown(P, _lib, peer_mod, ep, plan, ["pack", "forward", "backward_grad", "backward",
                                                                 "combine", "loss"],
                                  I, T, t, st, flush, barrier, False, False)
            exchange = {"value": B / (fms / 1e3), "unit": UNIT, "ms_per_step": fms, "loss": x_loss,
                        "phases_ms": xph,
                        "backward_tflops": 8.0 * b * B * D / (xph["backward"] / 1e3) / 1e12,
                        "note": "DISCO_BACKWARD=exchange: intra + cross GEMMs (8*b*B*D backward flops), "
                                "the reference's dataflow; also bitwise N-invariant"}
        finally:
            if saved is None:
                os.environ.pop("DISCO_BACKWARD", None)
            else:
                os.environ["DISCO_BACKWARD"] = saved

    # NVML's throttle reasons lag a ~50 ms burst: sample over ~0.5 s more of the same work (untimed,
    # after every measurement) so a power cap that shaped the timed steps is reported
    with ClockSampler(local_rank) as clk_after:
        for _ in range(max(20, 100 // max(1, args.steps))):
            step()
        torch.cuda.synchronize()
    P.finish_status(plan)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline ----------------------------------------------------------
    burst, sustained, hbm, src = load_peaks()
    mm = 4.0 * b * B * D           # 2 directions x 2*b*B*D (12*b*B*D per step)
    g_bytes = 2.0 * b * B * 2       # f16 E / G blocks (a6 output, both directions)
    recompute = phases.get("backward_grad", 0.0) > 0.1  # non-canonical shapes recompute the logits
    kernels = {  # name: (ms, bound, algorithmic work per launch, unit, peak)
        "logits_fwd": (phases["forward"], "tensor", mm, "TFLOP/s", sustained)}
    if recompute:
        kernels["logits_grad"] = (phases["backward_grad"], "hbm", g_bytes, "GB/s", hbm)
    # dual backward: one GEMM per gradient on H = G_d + G_d'^T, 4*b*B*D executed flops for the
    # reference's 8*b*B*D; the roofline uses the executed flops
    if dual or world == 1:
        kernels["gemm_backward"] = (phases["backward"], "tensor", (1 if dual else 2) * mm, "TFLOP/s", sustained)
    elif use_peer:
        kernels["gemm_backward_peer"] = (phases["backward_peer"], "tensor", 2 * mm, "TFLOP/s", sustained)
    else:
        kernels["gemm_cross"] = (phases["backward_cross"], "tensor", mm, "TFLOP/s", sustained)
        kernels["gemm_intra"] = (phases["backward_intra"], "tensor", mm, "TFLOP/s", sustained)
    table = {}
    for k, (kms, bound, work, unit, peak) in kernels.items():
        scale = 1e12 if unit == "TFLOP/s" else 1e9
        ach = work / (kms / 1e3) / scale
        table[k] = {"ms": kms, "bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                    "frac_of_burst": ach / burst if unit == "TFLOP/s" else None}
    # the forward also streams the f16 E blocks out (canonical shapes): its HBM side
    table["logits_fwd"]["e_write_gbs"] = None if recompute else g_bytes / (phases["forward"] / 1e3) / 1e9
    if "combine" in phases and dual:  # reads the K-half partials + label rows, writes the fp32 gradients
        cb = 2 * b * D * 4 * 2 + 2 * b * D * 4 + 2 * b * D * 2
        table["combine_dual"] = {"ms": phases["combine"], "bound": "hbm", "achieved": cb / (phases["combine"] / 1e3) / 1e9,
                                 "peak": hbm, "unit": "GB/s", "frac": cb / (phases["combine"] / 1e3) / 1e9 / hbm,
                                 "bytes": cb}
    dom = max((k for k in table if table[k]["unit"] == "TFLOP/s"), key=lambda k: table[k]["ms"])
    # ncu DRAM bytes per launch were captured at the headline workload (B=32K, D=512, N=1)
    traffic = load_traffic().get(dom) if (B, D, world) == (B_GLOBAL, DIM, 1) else None
    if "gemm_backward" in table and not recompute:  # E read once per gradient GEMM (dual) or twice
        table["gemm_backward"]["e_read_gbs"] = (1 if dual else 2) * g_bytes / (phases["backward"] / 1e3) / 1e9
    if dual:
        table["gemm_backward"]["algorithmic_tflops"] = 2 * mm / (phases["backward"] / 1e3) / 1e12
        table["gemm_backward"]["note"] = ("dual backward: H = G_d + G_d'^T formed in shared memory from the rank's own "
                                          "E block, 4*b*B*D executed flops (the reference's algorithm: 8*b*B*D)")
    step_tflops = 12.0 * b * B * D / (ms / 1e3) / 1e12            # algorithmic
    step_exec_tflops = (8.0 if dual else 12.0) * b * B * D / (ms / 1e3) / 1e12
    d = table[dom]

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        I_c, T_c = cpu_features(B, D)
        kind = reference_kind(args)
        if kind == "reference":
            sec = unmodified_reference_step(I_c, T_c, world)
            sample = (f"one full step: unmodified reference disco_step via run_ranks(lockstep), verification on, "
                      f"{b} rows x {B} columns, D={D}, f32, {cpu_cores()} cores ({sec:.1f} s)")
        else:
            sec = cpu_port_step(I_c, T_c, world)
            sample = (f"one full step: {b} rows x {B} columns, D={D}, both directions "
                      f"(oracle.disco_step_blocked, f32, {cpu_cores()} threads; {sec:.1f} s)")
        cpu = {"value": B / sec, "unit": UNIT, "cores": cpu_cores(), "kind": kind, "sample": sample}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": dict(workload_config(args, B, D, world),
                       backward="dual (rank-local H = G_d + G_d'^T GEMMs)" if dual else "exchange (intra + cross GEMMs)",
                       exchange=("none" if world == 1 else
                                 ("peer all-gather + nccl stats all_gather" if use_peer else
                                  "nccl all_gather (features, stats)") if dual else
                                 "peer (GEMM epilogue TMA pushes over NVLink)" if use_peer else "nccl all_to_all"),
                       exchange_preflight=preflight,
                       l2="flushed between steps (512 MB write, outside timed events)"),
        "loss": loss,
        "peak_loss_mem_gb": (loss_mem + peer_bytes) / 1e9,
        "loss_mem_detail": {"e_blocks_gb": g_bytes_ws / 1e9, "workspace_gb": plan.ws.numel() / 1e9,
                            "peer_window_gb": peer_bytes / 1e9,
                            "reference_loss_scope_elems": 2 * b * B,
                            "note": "max_memory_allocated delta of the first step (workspace + outputs) + the "
                                    "peer window (cudaMalloc'd outside torch, N > 1 peer transport); "
                                    "E blocks = 2*b*B f16 = the reference's 2*b*B loss elements (costs.py:110-112)"},
        "exchange_traffic": traffic_n,
        "peak_mem_gb": peak_mem / 1e9,
        "roofline": {"bound": d["bound"], "kernel": dom, "achieved": d["achieved"], "peak": d["peak"],
                     "unit": d["unit"], "frac": d["frac"], "traffic": traffic,
                     "peak_kind": f"{src} ({'bf16 sustained' if d['unit'] == 'TFLOP/s' else 'HBM copy'})",
                     "launch_ms": d["ms"], "step_tflops_algorithmic": step_tflops,
                     "step_tflops": step_exec_tflops, "step_frac": step_exec_tflops / sustained,
                     "step_frac_of_burst": step_exec_tflops / burst, "kernels": table},
        "phases_ms": phases,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "exchange_backward": exchange,
        "gpu_launches": launches,
        "clocks": dict(clk.summary(), in_kernel_mhz=kernel_mhz,
                       reasons_sustained=clk_after.summary().get("reasons"),
                       in_kernel_note="SM clock the tensor-core kernels actually ran at (clock64 / globaltimer "
                                      "stamps of CTA 0); below NVML's sm_mhz because the 1000 W cap "
                                      "(sw_power_cap) paces tensor-bound work, see reasons_sustained"),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    cb, cd = CONFIGS[args.config]
    args.batch = args.batch or cb
    args.dim = args.dim or cd
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
