"""GPU: the dual backward (disco_b200_path_info PATH_DUAL, the default disco_step backward).

Each rank's gradient is one GEMM per direction over its own E block on H = G_d + G_d'^T: the
column softmax G_d'[c, r] = exp2(y[r, c] - lse2_d'[c]) is rebuilt from the rank's own logits and
the all_gathered column statistics, so there is no gradient reduce-scatter.  The reference
reaches the same gradients through per-rank full-size contributions and all_reduce(AVG)
(shard.py:149-154, 199-208).  Checked here against the f64 oracle (the reference restated,
pinned by test_oracle_golden.py) at the contract tolerance 1e-3, including the sign-flip hook
and the exact-recompute fixup for rows whose E range cannot carry a column term.
"""

import numpy as np
import pytest
import torch

import paper_2304_08480_b200 as P
from paper_2304_08480_b200 import _lib
from paper_2304_08480_b200.shard import clear_plans, get_plan
from oracle import disco_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-3


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def run_sim(I, T, world, t, **kw):
    b = I.shape[0] // world
    Id, Td = dev(I), dev(T)

    def fn(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        return P.disco_step(ep, Id[rows], Td[rows], t, **kw)

    res = P.run_ranks(world, fn)
    return (torch.cat([r[0] for r in res]).cpu().numpy(), torch.cat([r[1] for r in res]).cpu().numpy(),
            [r[2] for r in res])


def errors(di, dt, loss, I, T, t):
    ri, rt, rl = O.clip_grad_full(I, T, t)
    return (O.max_rel_error(di, ri), O.max_rel_error(dt, rt), abs(loss - rl[0]) / abs(rl[0]))


@pytest.fixture(autouse=True)
def _default_backward(monkeypatch):
    monkeypatch.delenv("DISCO_BACKWARD", raising=False)
    yield
    clear_plans()


@pytest.mark.parametrize("B,D,t,corr", [(1024, 16, 100.0, False), (1024, 4, 100.0, False), (1024, 8, 100.0, True),
                                        (2048, 64, 100.0, True), (2048, 64, 100.0, False), (4096, 512, 100.0, True),
                                        (2048, 512, 1.0, False), (2048, 128, 50.0, True), (4096, 768, 100.0, True)])
def test_dual_vs_oracle(B, D, t, corr):
    """Canonical shapes over the temperature / dimension range the simulation of the E encoding
    covered (small D at t = 100 is where the row-offset E is stretched furthest for the column
    term); N = 1 and N = 4 give the same bytes."""
    assert _lib.path_info(B, D, 1) & _lib.PATH_DUAL
    I, T = O.synthetic_features(B, D, 5, correlated=corr)
    di, dt, loss = P.disco_step(None, dev(I), dev(T), t)
    di, dt = di.cpu().numpy(), dt.cpu().numpy()
    e = errors(di, dt, loss, I, T, t)
    assert max(e) < TOL, e
    si, st, sl = run_sim(I, T, 4, t)
    assert si.tobytes() == di.tobytes() and st.tobytes() == dt.tobytes() and sl[0] == loss


@pytest.mark.parametrize("N", [2, 4, 8])
def test_dual_sign_flip_hook(N):
    """flip_cross_rank_sign (shard.py:158-162): the column terms of rows outside the rank's slice
    change sign -- the oracle's disco_step_all with the hook; at N = 1 a no-op."""
    B, D, t = 8192, 256, 10.0
    I, T = O.synthetic_features(B, D, 6)
    di, dt, losses = run_sim(I, T, N, t, flip_cross_rank_sign=True)
    oi, ot, ol = O.disco_step_all(I, T, N, t, flip_cross_rank_sign=True)
    assert O.max_rel_error(di, oi) < TOL and O.max_rel_error(dt, ot) < TOL
    assert abs(losses[0] - ol) / ol < TOL
    di1, dt1, _ = run_sim(I, T, 1, t, flip_cross_rank_sign=True)
    ni, nt, _ = run_sim(I, T, 1, t)
    assert di1.tobytes() == ni.tobytes() and dt1.tobytes() == nt.tobytes()


def _adversarial(B, D, n_anti, seed):
    """Features clustered around one direction u, except n_anti texts at -u: those columns'
    statistics sit ~260 log2 units below the rows' group maxima at t = 100, so the
    row-offset E cannot represent their column softmax -- every row meeting such a column in one
    of its groups must be recomputed exactly by the fixup."""
    rng = np.random.default_rng(seed)
    u = rng.standard_normal(D)
    I = u + 0.3 * rng.standard_normal((B, D))
    T = u + 0.3 * rng.standard_normal((B, D))
    anti = rng.choice(B, n_anti, replace=False)
    T[anti] = -u + 0.3 * rng.standard_normal((n_anti, D))
    I = O.bf16_round(O.l2_normalize_rows(I)).astype(np.float64)
    T = O.bf16_round(O.l2_normalize_rows(T)).astype(np.float64)
    return I, T


@pytest.mark.parametrize("N", [1, 2])
def test_dual_fixup_recomputes_flagged_rows(N):
    B, D, t = 2048, 64, 100.0
    I, T = _adversarial(B, D, 16, 3)
    di, dt, losses = run_sim(I, T, N, t)
    fixed = sum(get_plan(B, D, N, r, torch.device("cuda", 0)).fixed_rows for r in range(N))
    assert fixed > 0, "the adversarial columns should have queued rows for the exact recompute"
    e = errors(di, dt, losses[0], I, T, t)
    assert max(e) < TOL, e
    if N == 2:
        d1 = run_sim(I, T, 1, t)
        assert d1[0].tobytes() == di.tobytes() and d1[1].tobytes() == dt.tobytes()


def test_dual_fixup_refreshes_pipelined_host_outputs():
    """Host (numpy) inputs at N = 1 take the row-block path whose blocks are copied to the host as
    they finish; rows fixed afterwards must reach the host copies too."""
    B, D, t = 2048, 64, 100.0
    I, T = _adversarial(B, D, 16, 4)
    hi, ht, hl = P.disco_step(None, I.astype(np.float32), T.astype(np.float32), t)
    di, dt, dl = P.disco_step(None, dev(I), dev(T), t)
    assert get_plan(B, D, 1, 0, torch.device("cuda", 0)).fixed_rows > 0
    assert np.array_equal(hi, di.cpu().numpy()) and np.array_equal(ht, dt.cpu().numpy()) and hl == dl


def test_dual_no_fixup_on_synthetic_features():
    """The bench / parity features (cli.py:103-105) never need the recompute at D = 512."""
    B, D = 8192, 512
    I, T = O.synthetic_features(B, D, 8)
    P.disco_step(None, dev(I), dev(T), 100.0)
    assert get_plan(B, D, 1, 0, torch.device("cuda", 0)).fixed_rows == 0


def test_dual_matches_exchange_backward_across_n(monkeypatch):
    """The two backwards agree within the contract at N = 1, 2, 8 (different roundings of the
    same sums), and the dual one is bitwise N-invariant."""
    B, D, t = 4096, 512, 100.0
    I, T = O.synthetic_features(B, D, 9)
    base = None
    for N in (1, 2, 8):
        di, dt, losses = run_sim(I, T, N, t)
        if base is None:
            base = (di, dt, losses[0])
        assert di.tobytes() == base[0].tobytes() and dt.tobytes() == base[1].tobytes()
    monkeypatch.setenv("DISCO_BACKWARD", "exchange")
    ei, et, el = run_sim(I, T, 2, t)
    assert O.max_rel_error(base[0], ei) < TOL and O.max_rel_error(base[1], et) < TOL and el[0] == base[2]


def _raw_pair(B, D, seed, adversarial=False):
    """Raw (unnormalised) tower outputs whose row-normalised versions are the loss features."""
    rng = np.random.default_rng(seed)
    if adversarial:
        I, T = _adversarial(B, D, 16, seed)
        scale = rng.uniform(0.5, 3.0, (B, 1))
        return I * scale, T * scale[::-1]
    return rng.standard_normal((B, D)) * 2.0, rng.standard_normal((B, D)) * 0.5


@pytest.mark.parametrize("N,adversarial", [(1, False), (2, False), (1, True), (2, True)])
def test_fused_tower_epilogue_matches_unfused_kernels(N, adversarial):
    """the combine with l2_normalize_rows_backward fused into it (one warp per
    row, disco_b200_finish_dual_l2norm) gives the same bits as disco_step followed by the separate
    normalisation-backward kernel -- also for rows the dual fixup recomputes."""
    from paper_2304_08480_b200 import towers
    B, D, t = 2048, 64, 100.0
    Ir, Tr = _raw_pair(B, D, 5, adversarial)
    raw_i, raw_t = dev(Ir), dev(Tr)
    I, _ = towers.l2_normalize_rows(raw_i)
    T, _ = towers.l2_normalize_rows(raw_t)
    b = B // N

    def fused(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        ri, rt = raw_i[rows].contiguous(), raw_t[rows].contiguous()
        dx_i, dx_t = torch.empty_like(ri), torch.empty_like(rt)
        nf = torch.zeros(1, dtype=torch.int32, device="cuda")
        _, _, plan = P.disco_step_async(ep, I[rows], T[rows], t, l2norm=(ri, rt, dx_i, dx_t, nf))
        loss = P.finish_status(plan)
        return dx_i, dx_t, loss, int(nf.item()), plan.fixed_rows

    def unfused(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        di, dt, loss = P.disco_step(ep, I[rows], T[rows], t)
        return (towers.l2_normalize_rows_backward(raw_i[rows].contiguous(), di),
                towers.l2_normalize_rows_backward(raw_t[rows].contiguous(), dt), loss)

    fr = P.run_ranks(N, fused)
    ur = P.run_ranks(N, unfused)
    if adversarial:
        assert sum(r[4] for r in fr) > 0, "expected rows queued for the fixup"
    for a, u in zip(fr, ur):
        assert a[3] == 0
        assert a[2] == u[2]
        assert a[0].cpu().numpy().tobytes() == u[0].cpu().numpy().tobytes()
        assert a[1].cpu().numpy().tobytes() == u[1].cpu().numpy().tobytes()


def test_fused_tower_epilogue_exchange_mode_and_validation(monkeypatch):
    """With DISCO_BACKWARD=exchange the call runs the exchange backward and then the separate
    normalisation kernel (equal to composing them by hand); malformed l2norm arguments raise
    ShapeError before any launch."""
    from paper_2304_08480_b200 import towers
    B, D, t = 2048, 64, 10.0
    Ir, Tr = _raw_pair(B, D, 11)
    raw_i, raw_t = dev(Ir), dev(Tr)
    I, _ = towers.l2_normalize_rows(raw_i)
    T, _ = towers.l2_normalize_rows(raw_t)
    monkeypatch.setenv("DISCO_BACKWARD", "exchange")
    dx_i, dx_t = torch.empty_like(raw_i), torch.empty_like(raw_t)
    nf = torch.zeros(1, dtype=torch.int32, device="cuda")
    _, _, plan = P.disco_step_async(P.SingleEndpoint(), I, T, t,
                                    l2norm=(raw_i, raw_t, dx_i, dx_t, nf))
    P.finish_status(plan)
    di, dt, _ = P.disco_step(None, I, T, t)
    assert torch.equal(dx_i, towers.l2_normalize_rows_backward(raw_i, di))
    assert torch.equal(dx_t, towers.l2_normalize_rows_backward(raw_t, dt))
    monkeypatch.delenv("DISCO_BACKWARD")
    with pytest.raises(P.ShapeError):
        P.disco_step_async(P.SingleEndpoint(), I, T, t, l2norm=(raw_i[:, :32], raw_t, dx_i, dx_t, nf))
    with pytest.raises(P.ShapeError):
        P.disco_step_async(P.SingleEndpoint(), I, T, t, l2norm=(raw_i, raw_t, dx_i.double(), dx_t, nf))
    with pytest.raises(P.ShapeError):
        P.disco_step_async(P.SingleEndpoint(), I, T, t, l2norm=(raw_i, raw_t, dx_i, dx_t, nf.float()))


@pytest.mark.parametrize("N", [2, 4])
def test_host_outputs_at_n_gt_1_row_blocks_bitwise(N):
    """numpy inputs at N > 1 (dual path): each rank's gradients come back in row blocks whose copies
    overlap the next block's GEMM; same bytes as the device-tensor step."""
    B, D, t = 16384, 256, 100.0
    I, T = O.synthetic_features(B, D, 13)
    b = B // N
    Id, Td = dev(I), dev(T)

    def host(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        return P.disco_step(ep, I[rows].astype(np.float32), T[rows].astype(np.float32), t)

    def device(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        return P.disco_step(ep, Id[rows], Td[rows], t)

    hr = P.run_ranks(N, host)
    dr = P.run_ranks(N, device)
    for h, d in zip(hr, dr):
        assert isinstance(h[0], np.ndarray) and h[2] == d[2]
        assert np.array_equal(h[0], d[0].cpu().numpy()) and np.array_equal(h[1], d[1].cpu().numpy())
