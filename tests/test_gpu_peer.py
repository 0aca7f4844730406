"""GPU: the peer transport against the all_to_all path and N = 1.

Both backwards run over it: the default dual backward (the peer all-gather of the packed rows,
then only the row statistics are exchanged) and the exchange backward (DISCO_BACKWARD=exchange),
whose backward GEMM pushes every cross tile into the owner's peer window (TMA stores through
per-destination tensor maps), a one-warp kernel publishes an arrival epoch, and the owner's
combine waits for all N epochs.  Results must be bit-identical to the NCCL-style path (same
fixed tree, evaluated at the owner), to N = 1, and must stay so across steps (the two parity
windows alternate).

Simulated ranks are threads on one GPU, each on its own stream (the wait kernel spins on device
flags, so ranks must progress independently).  The two-process test runs two real processes on
the same GPU over gloo with CUDA IPC-mapped windows: the cross-process mapping, tensor maps on
IPC pointers and the system-scope flag protocol, everything but NVLink itself.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_2304_08480_b200 as P
from oracle import disco_oracle as O

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def sim(I, T, N, t, peer, steps=1, **kw):
    b = I.shape[0] // N
    Id, Td = dev(I), dev(T)

    def fn(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        out = None
        for _ in range(steps):
            out = P.disco_step(ep, Id[rows], Td[rows], t, **kw)
        return out

    res = P.run_ranks(N, fn, peer=peer, own_streams=True)
    di = torch.cat([r[0] for r in res]).cpu().numpy()
    dt = torch.cat([r[1] for r in res]).cpu().numpy()
    return di, dt, [r[2] for r in res]


@pytest.mark.parametrize("backward", ["dual", "exchange"])
@pytest.mark.parametrize("B,D", [(4096, 512), (2048, 768), (3072, 256)])
def test_peer_matches_all_to_all_and_single_rank(B, D, monkeypatch, backward):
    monkeypatch.setenv("DISCO_BACKWARD", backward)
    I, T = O.synthetic_features(B, D, 7)
    di1, dt1, l1 = P.disco_step(None, dev(I), dev(T), 100.0)
    di1, dt1 = di1.cpu().numpy(), dt1.cpu().numpy()
    Ns = [2, 4, 8] if B % 1024 == 0 and (B // 8) % 128 == 0 else [2]
    for N in Ns:
        if (B // N) % 128:
            continue
        pi, pt, pl = sim(I, T, N, 100.0, peer=True, steps=3)  # parity windows alternate
        ai, at, al = sim(I, T, N, 100.0, peer=False)
        assert pi.tobytes() == ai.tobytes() and pt.tobytes() == at.tobytes(), f"peer != all_to_all at N={N}"
        assert len(set(pl)) == 1 and pl[0] == al[0]
        if B % 1024 == 0:  # canonical chunking: equal to N = 1 bit for bit
            assert pi.tobytes() == di1.tobytes() and pt.tobytes() == dt1.tobytes() and pl[0] == l1
    ri, rt, _ = O.clip_grad_full(O.bf16_round(I), O.bf16_round(T), 100.0)
    assert O.max_rel_error(di1, ri) < 1e-3 and O.max_rel_error(dt1, rt) < 1e-3


@pytest.mark.parametrize("backward", ["dual", "exchange"])
def test_peer_sign_flip_matches_all_to_all(monkeypatch, backward):
    monkeypatch.setenv("DISCO_BACKWARD", backward)
    B, D = 2048, 256
    I, T = O.synthetic_features(B, D, 8)
    pi, pt, _ = sim(I, T, 2, 10.0, peer=True, flip_cross_rank_sign=True)
    ai, at, _ = sim(I, T, 2, 10.0, peer=False, flip_cross_rank_sign=True)
    assert pi.tobytes() == ai.tobytes() and pt.tobytes() == at.tobytes()


@pytest.fixture(autouse=True)
def _release_windows():
    yield
    from paper_2304_08480_b200.shard import clear_plans
    clear_plans()


def test_peer_missing_rank_times_out_instead_of_hanging(monkeypatch):
    """An epoch that never arrives: the wait kernels give up and both hosts raise."""
    from paper_2304_08480_b200 import peer as peer_mod
    from paper_2304_08480_b200.shard import get_plan

    monkeypatch.setattr(peer_mod, "PEER_TIMEOUT_S", 0.5)
    monkeypatch.setenv("DISCO_BACKWARD", "exchange")
    B, D = 2048, 256
    I, T = O.synthetic_features(B, D, 9)
    Id, Td = dev(I), dev(T)

    def fn(ep):
        rows = slice(ep.rank * 1024, (ep.rank + 1) * 1024)
        P.disco_step(ep, Id[rows], Td[rows], 10.0)  # both ranks: epoch 1
        if ep.rank == 1:  # rank 1 skips an epoch: the ranks wait for epochs the other never sends
            get_plan(B, D, 2, 1, Id.device).peer_window(ep).next_step()
        with pytest.raises(P.CollectiveTimeoutError):
            P.disco_step(ep, Id[rows], Td[rows], 10.0)
        return None

    P.run_ranks(2, fn, peer=True, own_streams=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode,streamed,backward", [("peer", "0", "dual"), ("peer", "1", "dual"), ("nccl", "0", "dual"),
                                                    ("fallback", "0", "dual"), ("peer", "0", "exchange"),
                                                    ("nccl", "0", "exchange")])
def test_peer_two_processes_ipc(tmp_path, monkeypatch, mode, streamed, backward):
    """Two processes, one GPU, gloo: bitwise equal to N = 1.  ``peer``: CUDA IPC windows, with the
    kernel all-gather and (small B, where the shared GPU's time slicing lets both ranks publish
    before either spins for long) the streamed copy-engine all-gather.  ``nccl``: DISCO_PEER=0, the
    ProcessGroupEndpoint all_gather / all_to_all exchange (shard.py:190-205 replaced by
    fabric.py all_gather_into + all_to_all_into) driving the real kernels, host-staged.
    ``fallback``: peer requested but unavailable (access check fails on every rank): both ranks
    drop to the NCCL exchange instead of hanging."""
    B, D = 2048, 256
    I, T = O.synthetic_features(B, D, 11)
    np.save(tmp_path / "I.npy", I.astype(np.float32))
    np.save(tmp_path / "T.npy", T.astype(np.float32))
    port = _free_port()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2",
               DISCO_PEER_STREAMED=streamed, DISCO_PEER_TIMEOUT="30", DISCO_PEER="0" if mode == "nccl" else "1",
               DISCO_BACKWARD=backward)
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "peer_worker.py"), str(tmp_path), mode],
                                      env=e))
    rcs = []
    for p in procs:
        try:
            rcs.append(p.wait(timeout=240))
        except subprocess.TimeoutExpired:
            p.kill()
            rcs.append("timeout")
    assert rcs == [0, 0], rcs
    monkeypatch.setenv("DISCO_BACKWARD", backward)
    di1, dt1, l1 = P.disco_step(None, dev(I), dev(T), 100.0)
    got_i = np.concatenate([np.load(tmp_path / f"di{r}.npy") for r in range(2)])
    got_t = np.concatenate([np.load(tmp_path / f"dt{r}.npy") for r in range(2)])
    losses = [float(np.load(tmp_path / f"loss{r}.npy")) for r in range(2)]
    assert got_i.tobytes() == di1.cpu().numpy().tobytes()
    assert got_t.tobytes() == dt1.cpu().numpy().tobytes()
    assert losses[0] == losses[1] == l1
