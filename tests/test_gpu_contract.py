"""Contracts at the public entry points, on the device path.

  * Counters through ``local_loss_and_grads`` and ``disco_step`` (test_shard.py:172-185,
    test_costs.py:165-171): loss peak 2*b*B, loss FLOPs 4*b*B*D, exchange peak 2*B*D inside
    local_loss_and_grads and 5*B*D inside disco_step, exchange FLOPs 8*b*B*D.
  * ``costs.measured_detail`` keeps the reference tuple (loss_peak, loss_flops, exchange_peak)
    and reproduces the reference's own outputs (tests/golden/reference_towers.npz "measured").
  * The plan cache does not grow with fresh rank threads.
  * ``disco_step_async`` rejects inputs the kernels cannot read safely, before any launch.
"""

import os

import numpy as np
import pytest
import torch

import paper_2304_08480_b200 as P
from paper_2304_08480_b200 import costs, shard
from paper_2304_08480_b200.counters import Counters
from oracle import disco_oracle as O

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_towers.npz")


def test_local_loss_and_grads_counters():
    """test_shard.py:172-185."""
    batch, dim, world = 8, 4, 2
    local = batch // world
    I, T = O.synthetic_features(batch, dim, 7)
    lc, xc = Counters(), Counters()
    P.local_loss_and_grads(P.ShardLayout(world_size=world, global_batch=batch, rank=0), I, T, 10.0,
                           loss_counters=lc, exchange_counters=xc)
    assert lc.peak_live_elements == 2 * local * batch
    assert lc.live_elements == 0
    assert lc.flops == 4 * local * batch * dim
    assert xc.peak_live_elements == 2 * batch * dim
    assert xc.flops == 8 * local * batch * dim


@pytest.mark.parametrize("world", [1, 2, 4])
def test_disco_step_counters(world):
    """disco_step's exchange scope peaks at 5*B*D (test_costs.py:165-171); the loss scope is the
    local_loss_and_grads accounting of each rank."""
    B, D = 32, 4
    b = B // world
    I, T = O.synthetic_features(B, D, 1)
    Id = torch.from_numpy(I.astype(np.float32)).cuda()
    Td = torch.from_numpy(T.astype(np.float32)).cuda()

    def fn(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        lc, xc = Counters(), Counters()
        P.disco_step(ep, Id[rows], Td[rows], 10.0, loss_counters=lc, exchange_counters=xc)
        return lc, xc

    for lc, xc in P.run_ranks(world, fn):
        assert lc.peak_live_elements == 2 * b * B and lc.live_elements == 0
        assert lc.flops == 4 * b * B * D
        assert xc.peak_live_elements == 5 * B * D
        assert xc.flops == 8 * b * B * D


def test_measured_detail_matches_the_reference_outputs():
    """costs.measured_detail(mode, B, N, D) == the reference's (loss_peak, loss_flops, exchange_peak)
    for every case tests/golden/gen_golden_towers.py recorded from the reference itself."""
    rows = np.load(GOLDEN)["measured"]
    assert len(rows) >= 8
    for is_disco, B, N, D, lp, lf, xp in rows.tolist():
        got = costs.measured_detail("disco" if is_disco else "naive", B, N, D)
        assert got == (lp, lf, xp), (is_disco, B, N, D, got, (lp, lf, xp))


def test_measured_detail_validation():
    with pytest.raises(P.DomainError):
        costs.measured_detail("fused", 16, 1, 4)
    with pytest.raises(P.DomainError):
        costs.measured_detail("naive", 16, 1, 4, precision="f16")
    with pytest.raises(P.DomainError):
        costs.measured_detail("disco", 16, 3, 4)
    with pytest.raises(P.DomainError):
        costs.measured_detail("disco", 16, 2, 4, scheduler="random")
    a = costs.measured_detail("disco", 64, 4, 8, scheduler="lockstep")
    c = costs.measured_detail("disco", 64, 4, 8, scheduler="concurrent")
    assert a == c


def test_plan_cache_is_shared_by_fresh_rank_threads():
    """Repeated run_ranks calls (new threads each time, as the reference's verify harness drives
    disco_step) reuse one workspace per (geometry, rank) instead of allocating a new one."""
    shard.clear_plans()
    I, T = O.synthetic_features(256, 64, 2)
    Id = torch.from_numpy(I.astype(np.float32)).cuda()
    Td = torch.from_numpy(T.astype(np.float32)).cuda()

    def fn(ep):
        rows = slice(ep.rank * 64, (ep.rank + 1) * 64)
        return P.disco_step(ep, Id[rows], Td[rows], 10.0)[2]

    first = P.run_ranks(4, fn)
    n = shard.cached_plans()
    assert n == 4
    for _ in range(5):
        assert P.run_ranks(4, fn) == first
    assert shard.cached_plans() == n
    # own streams per rank thread: the plans are reused across streams, ordered by events
    for _ in range(3):
        assert P.run_ranks(4, fn, own_streams=True) == first
    assert shard.cached_plans() == n
    shard.clear_plans()


def test_plan_cache_is_bounded(monkeypatch):
    shard.clear_plans()
    monkeypatch.setenv("DISCO_PLAN_CACHE_BYTES", str(1))  # every new geometry evicts the others
    for B in (64, 128, 256):
        I, T = O.synthetic_features(B, 32, 0)
        P.disco_step(None, torch.from_numpy(I.astype(np.float32)).cuda(),
                     torch.from_numpy(T.astype(np.float32)).cuda(), 10.0)
        assert shard.cached_plans() == 1
    shard.clear_plans()


def test_disco_step_async_rejects_unsafe_inputs():
    ep = P.SingleEndpoint()
    a = torch.randn(64, 32, device="cuda")
    with pytest.raises(P.ShapeError):
        P.disco_step_async(ep, a, torch.randn(32, 32, device="cuda"), 10.0)  # shapes disagree
    with pytest.raises(TypeError):
        P.disco_step_async(ep, a, a.to(torch.bfloat16), 10.0)  # dtypes disagree
    with pytest.raises(TypeError):
        P.disco_step_async(ep, a.to(torch.int32), a.to(torch.int32), 10.0)
    wide = torch.randn(32, 64, device="cuda")
    with pytest.raises(P.ShapeError):
        P.disco_step_async(ep, wide.t(), wide.t(), 10.0)  # column stride != 1
    with pytest.raises(P.ShapeError):
        P.disco_step_async(ep, a[None], a[None], 10.0)
    # a valid strided view (unit column stride, row stride > D) is read in place
    big = torch.nn.functional.normalize(torch.randn(64, 48, device="cuda"), dim=1).bfloat16().float()
    view = big[:, :32]
    d_i, d_t, plan = P.disco_step_async(ep, view, view, 10.0)
    loss = P.finish_status(plan)
    ri, rt, rl = O.clip_grad_full(view.double().cpu().numpy(), view.double().cpu().numpy(), 10.0)
    assert abs(loss - rl[0]) < 1e-3 * rl[0]
    assert O.max_rel_error(d_i.cpu().numpy(), ri) < 1e-3


def test_autograd_accepts_non_contiguous_features():
    base = torch.nn.functional.normalize(torch.randn(2, 128, 64, device="cuda"), dim=2).bfloat16().float()
    I = base[0].t().contiguous().t()  # column-major view (bf16-representable values, as the kernels see them)
    T = base[1]
    I.requires_grad_(True)
    loss = P.disco_loss(I, T, 10.0)
    loss.backward()
    ri, _, rl = O.clip_grad_full(I.detach().double().cpu().numpy(), T.double().cpu().numpy(), 10.0)
    assert abs(float(loss.detach()) - rl[0]) < 1e-3 * rl[0]
    assert O.max_rel_error(I.grad.cpu().numpy(), ri) < 1e-3
