"""GPU: the autograd wrapper -- loss, feature gradients and dL/dlogit_scale.

dL/dt has no reference counterpart; it is checked against
oracle.dlogit_scale_full, itself pinned by finite differences of the
reference-pinned clip_loss_full (tests/test_oracle_golden.py).
"""

import numpy as np
import pytest
import torch

import paper_2304_08480_b200 as P
from oracle import disco_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _feats(B, D, seed, correlated=False):
    I, T = O.synthetic_features(B, D, seed, correlated=correlated)  # bf16-rounded values
    return I, T


@pytest.mark.parametrize("B,D,t,corr", [(1024, 512, 100.0, False), (2048, 256, 14.2857, True), (96, 40, 10.0, False)])
def test_loss_and_all_grads_vs_oracle(B, D, t, corr):
    I, T = _feats(B, D, 11, corr)
    Id = torch.tensor(I, dtype=torch.float32, device="cuda", requires_grad=True)
    Td = torch.tensor(T, dtype=torch.float32, device="cuda", requires_grad=True)
    scale = torch.tensor(t, dtype=torch.float32, device="cuda", requires_grad=True)
    loss = P.disco_loss(Id, Td, scale)
    loss.backward()
    ri, rt, rl = O.clip_grad_full(I, T, t)
    rs = O.dlogit_scale_full(I, T, t)
    assert abs(loss.item() - rl[0]) / abs(rl[0]) < TOL
    assert O.max_rel_error(Id.grad.cpu().numpy(), ri) < TOL
    assert O.max_rel_error(Td.grad.cpu().numpy(), rt) < TOL
    assert abs(scale.grad.item() - rs) <= TOL * max(abs(rs), 1e-3), (scale.grad.item(), rs)


def test_bf16_features_get_bf16_grads_and_chain_rule():
    B, D = 1024, 128
    I, T = _feats(B, D, 5)
    Id = torch.tensor(I, device="cuda").bfloat16().requires_grad_(True)
    Td = torch.tensor(T, device="cuda").bfloat16().requires_grad_(True)
    log_scale = torch.tensor(np.log(50.0), dtype=torch.float32, device="cuda", requires_grad=True)
    loss = 3.0 * P.DiscoCLIPLoss()(Id, Td, log_scale.exp())
    loss.backward()
    assert Id.grad.dtype == torch.bfloat16 and Td.grad.dtype == torch.bfloat16
    ri, rt, _ = O.clip_grad_full(I, T, 50.0)
    # bf16 gradient output: 2^-9 relative rounding on top of the 1e-3 contract
    assert O.max_rel_error(Id.grad.float().cpu().numpy(), 3.0 * ri) < 5e-3
    rs = O.dlogit_scale_full(I, T, 50.0) * 50.0 * 3.0  # d/dlog_scale = t * dL/dt
    assert abs(log_scale.grad.item() - rs) <= TOL * abs(rs)


@pytest.mark.parametrize("peer", [False, True])
def test_dlogit_bitwise_identical_across_world_sizes(peer):
    """Loss, dL/dt and both feature gradients through autograd are the same bytes at N = 1, 2, 4, 8,
    with the NCCL-style exchange and with the peer transport (windows shared between the rank
    threads, one stream per rank)."""
    B, D, t = 2048, 64, 100.0
    I, T = _feats(B, D, 9)
    Id = torch.tensor(I, dtype=torch.float32, device="cuda")
    Td = torch.tensor(T, dtype=torch.float32, device="cuda")
    results = {}
    for N in (1, 2, 4, 8):
        b = B // N

        def fn(ep):
            rows = slice(ep.rank * b, (ep.rank + 1) * b)
            s = torch.tensor(t, device="cuda", requires_grad=True)
            Ir = Id[rows].clone().requires_grad_(True)
            Tr = Td[rows].clone().requires_grad_(True)
            loss = P.disco_loss(Ir, Tr, s, ep)
            loss.backward()
            return loss.item(), s.grad.item(), Ir.grad, Tr.grad

        res = P.run_ranks(N, fn, peer=peer and N > 1)
        assert len({r[0] for r in res}) == 1 and len({r[1] for r in res}) == 1
        results[N] = (res[0][0], res[0][1], torch.cat([r[2] for r in res]).cpu(), torch.cat([r[3] for r in res]).cpu())
    base = results[1]
    for N in (2, 4, 8):
        assert results[N][0] == base[0] and results[N][1] == base[1], N
        assert torch.equal(results[N][2], base[2]) and torch.equal(results[N][3], base[3]), N
