"""GPU parity: the sm_100a DisCo path against the CPU oracle.

The oracle (oracle/disco_oracle.py, pinned to the reference by
test_oracle_golden.py) runs in f64 on the SAME bf16-rounded features the
device sees.  Contract tolerance (BASELINE.json north_star): loss and
gradients within 1e-3, measured with the reference's normwise max_rel_error
(matrix.py:147-162) composed as in cli.py:114-122.  Across world sizes that
divide 8 (with B % 1024 == 0) results must be bitwise identical.
"""

import math

import numpy as np
import pytest
import torch

import paper_2304_08480_b200 as P
from oracle import disco_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-3


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def run_sim(I, T, world, t, **kw):
    """Simulated ranks on one GPU (threads); returns stacked grads + the per-rank losses."""
    b = I.shape[0] // world
    Id, Td = dev(I), dev(T)

    def fn(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        return P.disco_step(ep, Id[rows], Td[rows], t, **kw)

    res = P.run_ranks(world, fn)
    di = torch.cat([r[0] for r in res]).cpu().numpy()
    dt = torch.cat([r[1] for r in res]).cpu().numpy()
    losses = [r[2] for r in res]
    return di, dt, losses


def errors(di, dt, loss, I, T, t):
    ri, rt, rl = O.clip_grad_full(I, T, t)
    return (O.max_rel_error(di, ri), O.max_rel_error(dt, rt),
            O.max_rel_error(np.array([loss]), np.array([rl[0]])))


def test_known_answer_orthonormal():
    eye = np.eye(2)
    di, dt, loss = P.disco_step(None, eye, eye, 1.0)
    assert abs(loss - math.log(1.0 + math.exp(-1.0))) < 1e-6
    ri, rt, _ = O.clip_grad_full(eye, eye, 1.0)
    assert O.max_rel_error(di, ri) < TOL and O.max_rel_error(dt, rt) < TOL


def test_known_answer_identical_rows():
    feats = np.tile(np.array([1.0, 0.0, 0.0]), (4, 1))
    _, _, loss = P.disco_step(None, feats, feats, 10.0)
    assert abs(loss - math.log(4.0)) < 1e-6


def test_known_answer_single_pair():
    di, dt, loss = P.disco_step(None, np.array([[1.0, 0.0]]), np.array([[0.6, 0.8]]), 10.0)
    assert loss == 0.0
    assert not np.any(di) and not np.any(dt)


@pytest.mark.parametrize("B,D,N", [(8, 4, 1), (8, 5, 2), (12, 5, 3), (16, 8, 4), (64, 16, 8), (32, 8, 4)])
@pytest.mark.parametrize("t", [1.0, 10.0, 100.0])
def test_small_grid_vs_oracle(B, D, N, t):
    I, T = O.synthetic_features(B, D, 0)
    di, dt, losses = run_sim(I, T, N, t)
    assert len(set(losses)) == 1
    e = errors(di, dt, losses[0], I, T, t)
    assert max(e) < TOL, e


@pytest.mark.parametrize("correlated", [False, True])
@pytest.mark.parametrize("t", [14.2857, 100.0])
def test_config_a(t, correlated):
    I, T = O.synthetic_features(1024, 512, 0, correlated=correlated)
    di, dt, losses = run_sim(I, T, 2, t)
    e = errors(di, dt, losses[0], I, T, t)
    assert max(e) < TOL, e


@pytest.mark.parametrize("B,D", [(4096, 512), (2048, 768), (2048, 1024), (1000, 100)])
def test_single_gpu_vs_oracle(B, D):
    I, T = O.synthetic_features(B, D, 1)
    di, dt, loss = P.disco_step(None, dev(I), dev(T), 100.0)
    e = errors(di.cpu().numpy(), dt.cpu().numpy(), loss, I, T, 100.0)
    assert max(e) < TOL, e


@pytest.mark.parametrize("backward", ["dual", "exchange"])
def test_bitwise_identical_across_world_sizes(monkeypatch, backward):
    """N-invariance of both backwards (the default dual one and DISCO_BACKWARD=exchange)."""
    monkeypatch.setenv("DISCO_BACKWARD", backward)
    B, D, t = 8192, 512, 100.0
    I, T = O.synthetic_features(B, D, 2)
    base = None
    for N in (1, 2, 4, 8):
        di, dt, losses = run_sim(I, T, N, t)
        assert len(set(losses)) == 1
        if base is None:
            base = (di, dt, losses[0])
            e = errors(di, dt, losses[0], I, T, t)
            assert max(e) < TOL, e
        else:
            assert di.tobytes() == base[0].tobytes(), f"d_image differs at N={N}"
            assert dt.tobytes() == base[1].tobytes(), f"d_text differs at N={N}"
            assert losses[0] == base[2]


def test_repeat_runs_are_bitwise_identical():
    I, T = O.synthetic_features(2048, 512, 3)
    a = run_sim(I, T, 4, 10.0)
    b = run_sim(I, T, 4, 10.0)
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes() and a[2] == b[2]


@pytest.mark.parametrize("N", [2, 3, 4])
def test_local_contributions_vs_oracle(N):
    I, T = O.synthetic_features(96, 24, 4)
    parts = []
    for r in range(N):
        layout = P.ShardLayout(world_size=N, global_batch=96, rank=r)
        c = P.local_loss_and_grads(layout, I, T, 10.0)
        oi, ot, ol = O.local_loss_and_grads(N, r, I, T, 10.0)
        assert O.max_rel_error(c.d_image_full, oi) < TOL
        assert O.max_rel_error(c.d_text_full, ot) < TOL
        assert abs(c.local_loss - ol) / abs(ol) < TOL
        parts.append(c)
    ri, rt, rl = O.clip_grad_full(I, T, 10.0)
    assert O.max_rel_error(sum(p.d_image_full for p in parts) / N, ri) < TOL
    assert abs(sum(p.local_loss for p in parts) / N - rl[0]) < TOL * rl[0]


def test_sign_flip_hook():
    I, T = O.synthetic_features(64, 8, 0)
    di, dt, losses = run_sim(I, T, 2, 10.0, flip_cross_rank_sign=True)
    oi, ot, ol = O.disco_step_all(I, T, 2, 10.0, flip_cross_rank_sign=True)
    assert O.max_rel_error(di, oi) < TOL and O.max_rel_error(dt, ot) < TOL
    ri, _, _ = O.clip_grad_full(I, T, 10.0)
    assert O.max_rel_error(di, ri) > 1e-3
    di1, _, _ = run_sim(I, T, 1, 10.0, flip_cross_rank_sign=True)
    assert O.max_rel_error(di1, ri) < TOL  # no-op at N = 1


def test_nonfinite_input_raises():
    I, T = O.synthetic_features(16, 8, 0)
    I[3, 2] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        P.disco_step(None, I, T, 10.0)


def test_full_size_b32k_sampled_rows():
    """Config B at N=1 against the blocked f64 oracle on 64 sampled rows."""
    B, D, t = 32768, 512, 100.0
    I, T = O.synthetic_features(B, D, 0)
    di, dt, loss = P.disco_step(None, dev(I), dev(T), t)
    rows = np.linspace(0, B - 1, 64).astype(np.int64)
    ri, rt, rl = O.clip_grad_rows(I, T, t, rows)
    assert O.max_rel_error(di[rows].cpu().numpy(), ri) < TOL
    assert O.max_rel_error(dt[rows].cpu().numpy(), rt) < TOL
    assert abs(loss - rl[0]) / rl[0] < TOL


@pytest.fixture
def release_plans():
    yield
    from paper_2304_08480_b200.shard import clear_plans
    clear_plans()
    torch.cuda.empty_cache()


def test_config_c_bitwise_and_sampled_oracle(release_plans):
    """BASELINE config C (B=65536, D=768): N=8 simulated ranks == N=1 bitwise, sampled f64 oracle."""
    B, D, t = 65536, 768, 100.0
    I, T = O.synthetic_features(B, D, 5)
    d8 = run_sim(I, T, 8, t)
    from paper_2304_08480_b200.shard import clear_plans
    clear_plans()
    torch.cuda.empty_cache()
    di, dt, loss = P.disco_step(None, dev(I), dev(T), t)
    di, dt = di.cpu().numpy(), dt.cpu().numpy()
    assert di.tobytes() == d8[0].tobytes() and dt.tobytes() == d8[1].tobytes() and loss == d8[2][0]
    rows = np.linspace(0, B - 1, 32).astype(np.int64)
    ri, rt, rl = O.clip_grad_rows(I, T, t, rows)
    assert O.max_rel_error(di[rows], ri) < TOL
    assert O.max_rel_error(dt[rows], rt) < TOL
    assert abs(loss - rl[0]) / rl[0] < TOL


def test_large_index_space(release_plans):
    """b*B = 4.3e9 G elements per direction (> 2^31): 64-bit offsets, narrow (D=64) GEMM path."""
    B, D, t = 65536, 64, 14.2857
    I, T = O.synthetic_features(B, D, 6)
    di, dt, loss = P.disco_step(None, dev(I), dev(T), t)
    rows = np.array([0, 1, 4095, 32768, 54321, B - 1])
    ri, rt, rl = O.clip_grad_rows(I, T, t, rows, stats=O.clip_stats_blocked(I, T, t, block=4096))
    assert O.max_rel_error(di[rows].cpu().numpy(), ri) < TOL
    assert O.max_rel_error(dt[rows].cpu().numpy(), rt) < TOL
    assert abs(loss - rl[0]) / rl[0] < TOL


@pytest.mark.parametrize("B,D", [(4096, 512), (3072, 256), (2048, 768)])
def test_host_pipelined_readback_bitwise(B, D):
    """Host inputs at N=1 take the row-block pipelined backward (disco_b200_backward_rows +
    combine_rows, device->host copies overlapped); it must equal the device path bit for bit."""
    I, T = O.synthetic_features(B, D, 3)
    blocks = P.shard.row_blocks(B)
    assert blocks[0][0] == 0 and blocks[-1][1] == B
    dh_i, dh_t, lh = P.disco_step(None, I.astype(np.float32), T.astype(np.float32), 100.0)
    dd_i, dd_t, ld = P.disco_step(None, dev(I), dev(T), 100.0)
    assert isinstance(dh_i, np.ndarray) and dh_i.dtype == np.float32
    assert lh == ld
    assert np.array_equal(dh_i, dd_i.cpu().numpy()) and np.array_equal(dh_t, dd_t.cpu().numpy())
    ri, rt, _ = O.clip_grad_full(O.bf16_round(I), O.bf16_round(T), 100.0)
    assert O.max_rel_error(dh_i, ri) < TOL and O.max_rel_error(dh_t, rt) < TOL


@pytest.mark.parametrize("B,D,dtype", [(32768, 512, torch.bfloat16), (8192, 1024, torch.float32),
                                       (2048, 64, torch.float16), (4096, 200, torch.float64)])
def test_host_pipelined_forward_bitwise(B, D, dtype):
    """Host features at N=1 with B % 2048 == 0 take the wavefront forward (chunked H2D on a copy
    stream, disco_b200_pack_rows + forward_wave per landed chunk on two compute streams,
    forward_finish); pinned torch inputs, outputs equal to the device path bit for bit."""
    assert P.shard.host_pipelined(1, B, D)
    I, T = O.synthetic_features(B, D, 4)
    Ih = torch.from_numpy(I.astype(np.float32)).to(dtype).pin_memory()
    Th = torch.from_numpy(T.astype(np.float32)).to(dtype).pin_memory()
    for _ in range(2):  # second call reuses the plan, streams and pinned buffers
        dh_i, dh_t, lh = P.disco_step(None, Ih, Th, 100.0)
    dd_i, dd_t, ld = P.disco_step(None, Ih.cuda(), Th.cuda(), 100.0)
    assert not dh_i.is_cuda and lh == ld
    assert torch.equal(dh_i, dd_i.cpu()) and torch.equal(dh_t, dd_t.cpu())


def test_host_pipelined_nonfinite_in_late_chunk():
    """A NaN landing with the last H2D chunk is still flagged (the status reset is ordered before
    every wave's pack on both compute streams)."""
    B, D = 4096, 128
    I, T = O.synthetic_features(B, D, 2)
    T = T.astype(np.float32)
    T[B - 3, 7] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        P.disco_step(None, I.astype(np.float32), T, 10.0)
    di, dt, loss = P.disco_step(None, I.astype(np.float32), O.synthetic_features(B, D, 2)[1].astype(np.float32), 10.0)
    assert np.isfinite(loss)


def test_config_e_bitwise_and_sampled_oracle(release_plans, monkeypatch):
    """BASELINE config E (B=16384, D=1024: the non-distributed CLIP loss on one GPU): the
    default (dual) path at N=1 equals N=8 simulated ranks bit for bit; it and the exchange
    backward match the f64 oracle on sampled rows within 1e-3."""
    B, D, t = 16384, 1024, 100.0
    I, T = O.synthetic_features(B, D, 12)
    d8 = run_sim(I, T, 8, t)
    from paper_2304_08480_b200.shard import clear_plans
    clear_plans()
    rows = np.linspace(0, B - 1, 48).astype(np.int64)
    ri, rt, rl = O.clip_grad_rows(I, T, t, rows)
    for backward in ("dual", "exchange"):
        monkeypatch.setenv("DISCO_BACKWARD", backward)
        di, dt, loss = P.disco_step(None, dev(I), dev(T), t)
        di, dt = di.cpu().numpy(), dt.cpu().numpy()
        if backward == "dual":
            assert di.tobytes() == d8[0].tobytes() and dt.tobytes() == d8[1].tobytes() and loss == d8[2][0]
        assert O.max_rel_error(di[rows], ri) < TOL
        assert O.max_rel_error(dt[rows], rt) < TOL
        assert abs(loss - rl[0]) / rl[0] < TOL


def test_streamed_forward_missing_chunk_times_out():
    """The streamed forward's producers never wait unboundedly: a wave flag that is never raised
    sets status flag 16 and the host raises instead of the GPU hanging."""
    from paper_2304_08480_b200 import _lib
    from paper_2304_08480_b200.shard import get_plan
    B, D = 4096, 128
    plan = get_plan(B, D, 1, 0, torch.device("cuda", 0))
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("disco_b200_pack_rows", *plan.args, plan.feat.data_ptr(), plan.feat.data_ptr(), D, D, _lib.BF16, 1,
              0, 0, st)
    _lib.call("disco_b200_forward_streamed", *plan.args, 10.0, 0x7FFF0000, 0.2, st)  # epoch never signalled
    with pytest.raises(RuntimeError, match="never landed"):
        P.finish_status(plan)
    # the plan stays usable: a normal host-buffer step afterwards is correct
    I, T = O.synthetic_features(B, D, 13)
    Ih = torch.from_numpy(I.astype(np.float32)).bfloat16().pin_memory()
    Th = torch.from_numpy(T.astype(np.float32)).bfloat16().pin_memory()
    dh_i, dh_t, lh = P.disco_step(None, Ih, Th, 10.0)
    dd_i, dd_t, ld = P.disco_step(None, Ih.cuda(), Th.cuda(), 10.0)
    assert torch.equal(dh_i, dd_i.cpu()) and torch.equal(dh_t, dd_t.cpu()) and lh == ld


@pytest.mark.parametrize("B,D", [(4096, 512), (8192, 1024), (5120, 500), (4096, 1000)])
def test_dual_and_exchange_backwards_vs_oracle(B, D, monkeypatch):
    """The dual backward (default; one GEMM per gradient on H = G_d + G_d'^T over the rank's own
    E block) and the exchange backward (DISCO_BACKWARD=exchange; intra + cross GEMMs) are both
    within the contract tolerance of the f64 oracle and of each other; the host row-block path
    gives the device path's bytes; local_loss_and_grads (always the exchange form) equals the
    exchange step at N = 1; repeat runs are bitwise equal."""
    I, T = O.synthetic_features(B, D, 21)
    monkeypatch.setenv("DISCO_BACKWARD", "exchange")
    bi, bt, bl = P.disco_step(None, dev(I), dev(T), 100.0)
    bi, bt = bi.cpu().numpy(), bt.cpu().numpy()
    assert max(errors(bi, bt, bl, I, T, 100.0)) < TOL
    c = P.local_loss_and_grads(P.ShardLayout(world_size=1, global_batch=B, rank=0), I.astype(np.float32),
                               T.astype(np.float32), 100.0)
    assert np.array_equal(np.asarray(c.d_image_full, dtype=np.float32), bi)
    assert np.array_equal(np.asarray(c.d_text_full, dtype=np.float32), bt)
    monkeypatch.delenv("DISCO_BACKWARD")
    di, dt, loss = P.disco_step(None, dev(I), dev(T), 100.0)
    di, dt = di.cpu().numpy(), dt.cpu().numpy()
    assert not np.array_equal(di, bi)  # the dual path really ran (different rounding)
    assert max(errors(di, dt, loss, I, T, 100.0)) < TOL
    assert O.max_rel_error(di, bi) < 1e-3 and O.max_rel_error(dt, bt) < 1e-3 and loss == bl
    hi, ht, hl = P.disco_step(None, I.astype(np.float32), T.astype(np.float32), 100.0)
    assert np.array_equal(hi, di) and np.array_equal(ht, dt) and hl == loss
    ri, rt, rl = P.disco_step(None, dev(I), dev(T), 100.0)
    assert np.array_equal(ri.cpu().numpy(), di) and np.array_equal(rt.cpu().numpy(), dt) and rl == loss


def test_input_containers_and_dtypes_give_identical_bits():
    """The reference takes numpy float64 / float32 matrices (shard.py:169); the drop-in also takes
    torch tensors of any float dtype on the host or the device.  Features holding bf16 values are
    represented exactly by every one of them, so every container / dtype must give the same bits
    (numpy in -> numpy out in the input's float dtype, torch CUDA in -> CUDA out)."""
    B, D, t = 2048, 256, 50.0
    I, T = O.synthetic_features(B, D, 21)
    ref_i, ref_t, ref_l = P.disco_step(None, dev(I), dev(T), t)
    ref_i, ref_t = ref_i.cpu().numpy(), ref_t.cpu().numpy()
    cases = [
        (I.astype(np.float64), T.astype(np.float64)),
        (I.astype(np.float32), T.astype(np.float32)),
        (torch.from_numpy(I.astype(np.float32)), torch.from_numpy(T.astype(np.float32))),
        (torch.from_numpy(I).cuda(), torch.from_numpy(T).cuda()),
        (torch.from_numpy(I).cuda().bfloat16(), torch.from_numpy(T).cuda().bfloat16()),
        (torch.from_numpy(I.astype(np.float32)).pin_memory().bfloat16(),
         torch.from_numpy(T.astype(np.float32)).pin_memory().bfloat16()),
    ]
    for a, b in cases:
        di, dt, loss = P.disco_step(None, a, b, t)
        if isinstance(a, np.ndarray):
            assert isinstance(di, np.ndarray) and di.dtype == a.dtype
            di, dt = di.astype(np.float32), dt.astype(np.float32)
        else:
            di, dt = di.float().cpu().numpy(), dt.float().cpu().numpy()
        assert loss == ref_l, (type(a), getattr(a, "dtype", None))
        assert np.array_equal(di, ref_i) and np.array_equal(dt, ref_t), (type(a), getattr(a, "dtype", None))


@pytest.mark.parametrize("B,k0", [(32768, "12"), (16384, "0"), (16384, "5"), (16384, "16"), (8192, "-1")])
def test_split_host_schedule_bitwise(monkeypatch, B, k0):
    """The split host-buffer schedule (direction 1 inside the H2D wavefront with direction 0 of the
    first k0 waves, then direction 0 row block by row block with each block's d_image backward
    and copy, then the d_text blocks) returns the device path's bits for any k0."""
    from paper_2304_08480_b200 import shard
    calls = []
    real = shard._split_backward
    monkeypatch.setattr(shard, "_split_backward", lambda *a, **k: (calls.append(1), real(*a, **k)))
    monkeypatch.setenv("DISCO_SPLIT_K0", k0)
    D = 512
    I, T = O.synthetic_features(B, D, 6)
    Ih = torch.from_numpy(I.astype(np.float32)).to(torch.bfloat16).pin_memory()
    Th = torch.from_numpy(T.astype(np.float32)).to(torch.bfloat16).pin_memory()
    dh_i, dh_t, lh = P.disco_step(None, Ih, Th, 100.0)
    dd_i, dd_t, ld = P.disco_step(None, Ih.cuda(), Th.cuda(), 100.0)
    assert calls, "the split schedule was not taken"
    assert lh == ld
    assert torch.equal(dh_i, dd_i.cpu()) and torch.equal(dh_t, dd_t.cpu())


def test_split_host_schedule_refreshes_fixed_rows(monkeypatch):
    """Rows the dual fixup recomputes after their blocks were copied reach the host copies."""
    from paper_2304_08480_b200 import shard
    calls = []
    real = shard._split_backward
    monkeypatch.setattr(shard, "_split_backward", lambda *a, **k: (calls.append(1), real(*a, **k)))
    from paper_2304_08480_b200.shard import get_plan
    from tests.test_gpu_dual import _adversarial
    B, D, t = 4096, 64, 100.0
    I, T = _adversarial(B, D, 16, 3)
    Ih = torch.from_numpy(I.astype(np.float32)).to(torch.bfloat16).pin_memory()
    Th = torch.from_numpy(T.astype(np.float32)).to(torch.bfloat16).pin_memory()
    hi, ht, hl = P.disco_step(None, Ih, Th, t)
    di, dt, dl = P.disco_step(None, Ih.cuda(), Th.cuda(), t)
    assert calls
    assert get_plan(B, D, 1, 0, torch.device("cuda", 0)).fixed_rows > 0
    assert torch.equal(hi, di.cpu()) and torch.equal(ht, dt.cpu()) and hl == dl
