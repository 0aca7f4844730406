"""Collective backend on CPU: gloo world_size 2 processes and the threaded LocalGroup.

The B200 path issues its collectives through these endpoints (fabric.py); on a
GPU box the same calls run over NCCL.  Here gloo carries CPU tensors, and the
test-only exchange emulation (exchange_emulation.py) proves that the slab
layout, the all_to_all and the fixed reduction trees give results bitwise
identical across world sizes and equal to the oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2304_08480_b200 as P
from oracle import disco_oracle as O
from tests import exchange_emulation as E


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, I, T, t, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ep = P.ProcessGroupEndpoint()
        assert ep.rank == rank and ep.world_size == world
        # reference-compatible collectives (fabric.py:257-275)
        local = torch.full((2, 3), float(rank + 1), dtype=torch.float64)
        gathered = ep.all_gather(local)
        red = ep.all_reduce(gathered * 0.5, P.ReduceOp.AVG)
        scal = ep.all_reduce_scalar(0.1 * (rank + 1), "avg")
        ep.barrier()
        # the DisCo exchange over real collectives
        B = I.shape[0]
        b = B // world
        intra, send, ce = E.local_phase(rank, world, I, T, t)
        recv = torch.empty_like(torch.from_numpy(send))
        work = ep.all_to_all_into(recv.view(-1), torch.from_numpy(send).reshape(-1), async_op=True)
        work.wait()
        ce_all = torch.empty((world, 2, b), dtype=torch.float32)
        ep.all_gather_into(ce_all.view(-1), torch.from_numpy(ce).reshape(-1))
        gi, gt = E.owner_phase(rank, world, t, B, intra, recv.numpy())
        loss = E.loss_from(ce_all.numpy(), world, b)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), gathered=gathered.numpy(), red=red.numpy(),
                 scal=np.array([scal]), gi=gi, gt=gt, loss=np.array([loss]))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def problem():
    I, T = O.synthetic_features(1024, 16, 5)
    return I, T, 10.0


def test_gloo_world2_collectives_and_exchange(tmp_path, problem):
    I, T, t = problem
    world = 2
    mp.start_processes(_gloo_worker, args=(world, _free_port(), I, T, t, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    res = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    want_gather = np.concatenate([np.full((2, 3), 1.0), np.full((2, 3), 2.0)])
    for r in res:
        assert np.array_equal(r["gathered"], want_gather)
        assert r["red"].tobytes() == (want_gather * 0.5).tobytes()  # AVG of identical buffers
        assert r["scal"][0] == (0.1 + 0.2) / 2
    d_image = np.concatenate([r["gi"] for r in res])
    d_text = np.concatenate([r["gt"] for r in res])
    assert res[0]["loss"][0] == res[1]["loss"][0]
    # bitwise identical to the single-process N=1 and N=2 emulations
    for N in (1, 2):
        si, st, sl = E.run_single_process(N, I, T, t)
        assert si.tobytes() == d_image.tobytes() and st.tobytes() == d_text.tobytes()
        assert sl == res[0]["loss"][0]
    ri, rt, rl = O.clip_grad_full(I, T, t)
    assert O.max_rel_error(d_image, ri) < 1e-5 and O.max_rel_error(d_text, rt) < 1e-5
    assert abs(res[0]["loss"][0] - rl[0]) < 1e-5 * rl[0]


def test_emulated_exchange_is_bitwise_invariant_across_world_sizes(problem):
    I, T, t = problem
    base = E.run_single_process(1, I, T, t)
    for N in (2, 4, 8):
        got = E.run_single_process(N, I, T, t)
        assert got[0].tobytes() == base[0].tobytes(), N
        assert got[1].tobytes() == base[1].tobytes(), N
        assert got[2] == base[2]


def test_peer_transport_tree_is_bitwise_the_all_to_all_tree(problem):
    """Peer transport order (leaves pushed un-presummed, owner tree over N*np leaves) equals the
    all_to_all order (sender presum, owner tree over sources) bit for bit, at every N."""
    I, T, t = problem
    base = E.run_single_process(1, I, T, t)
    for N in (2, 4, 8):
        got = E.run_single_process_peer(N, I, T, t)
        assert got[0].tobytes() == base[0].tobytes(), N
        assert got[1].tobytes() == base[1].tobytes(), N
    I2, T2 = O.synthetic_features(96, 8, 1)  # non-canonical chunking (N chunks)
    for N in (2, 3):
        a = E.run_single_process(N, I2, T2, t)
        b = E.run_single_process_peer(N, I2, T2, t)
        assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()


def _exchange_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ep = P.ProcessGroupEndpoint(peer=True)
        got = ep.exchange(bytes([rank]) * 64)  # a peer-window IPC handle is 64 opaque bytes
        np.save(os.path.join(outdir, f"x{rank}.npy"), np.frombuffer(b"".join(got), dtype=np.uint8))
    finally:
        dist.destroy_process_group()


def test_gloo_handle_exchange(tmp_path):
    world = 2
    mp.start_processes(_exchange_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn")
    want = np.frombuffer(bytes([0]) * 64 + bytes([1]) * 64, dtype=np.uint8)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"x{r}.npy"), want)


def test_peer_transport_switch(monkeypatch):
    from paper_2304_08480_b200 import peer

    g = P.LocalGroup(2, peer=True)
    assert peer.enabled(g.endpoint(0))
    assert not peer.enabled(P.LocalGroup(2, peer=False).endpoint(1))
    assert not peer.enabled(P.LocalGroup(1, peer=True).endpoint(0))  # nothing to exchange at N = 1
    assert not peer.enabled(P.LocalGroup(4).endpoint(0))  # simulated ranks: opt-in

    class PG:  # a process-group endpoint without an explicit choice follows DISCO_PEER
        world_size, peer = 4, None

    monkeypatch.delenv("DISCO_PEER", raising=False)
    assert peer.enabled(PG())  # default: on
    monkeypatch.setenv("DISCO_PEER", "0")
    assert not peer.enabled(PG())
    assert peer.supported(32768, 512, 8, 0) and peer.supported(2048, 256, 2, 1)
    assert not peer.supported(32768, 512, 16, 0) and not peer.supported(1000, 512, 2, 0)
    assert not peer.supported(4096, 64, 64, 0)
    res = P.run_ranks(3, lambda ep: ep.exchange(ep.rank * 10))
    assert res == [[0, 10, 20]] * 3


def test_local_group_threads_on_cpu_tensors():
    def fn(ep):
        x = torch.full((1, 2), float(ep.rank))
        g = ep.all_gather(x)
        out = torch.empty(ep.world_size * 2)
        ep.all_gather_into(out, x.reshape(-1))
        a2a_in = torch.arange(ep.world_size, dtype=torch.float32) + 10 * ep.rank
        a2a_out = torch.empty_like(a2a_in)
        ep.all_to_all_into(a2a_out, a2a_in)
        red = ep.all_reduce(g + 1.0, P.ReduceOp.SUM)
        s = ep.all_reduce_scalar(float(ep.rank), P.ReduceOp.AVG)
        ep.barrier()
        return g, out, a2a_out, red, s

    world = 4
    res = P.run_ranks(world, fn, device=None)
    want = torch.arange(world, dtype=torch.float32).repeat_interleave(2).reshape(world, 2)
    for r, (g, out, a2a, red, s) in enumerate(res):
        assert torch.equal(g, want) and torch.equal(out, want.reshape(-1))
        assert a2a.tolist() == [10.0 * src + r for src in range(world)]
        assert torch.equal(red, (want + 1.0) * world)
        assert s == sum(range(world)) / world


def test_local_group_contract_error_and_propagation():
    def fn(ep):
        if ep.rank == 0:
            return ep.all_gather(torch.zeros(1, 2))
        return ep.all_reduce(torch.zeros(1, 2))

    with pytest.raises(P.CollectiveContractError):
        P.run_ranks(2, fn, device=None)

    def boom(ep):
        if ep.rank == 1:
            raise KeyError("rank 1 failed")
        ep.barrier()

    with pytest.raises(KeyError):
        P.run_ranks(2, boom, device=None)


def test_local_group_timeout_names_missing_rank():
    def fn(ep):
        if ep.rank == 0:
            ep.barrier()

    group = P.LocalGroup(2, timeout=0.5)
    import threading
    errs = []

    def w(r):
        try:
            if r == 0:
                group.endpoint(0).barrier()
        except Exception as exc:  # noqa: BLE001
            errs.append(exc)

    th = [threading.Thread(target=w, args=(r,)) for r in range(2)]
    [x.start() for x in th]
    [x.join() for x in th]
    assert len(errs) == 1 and isinstance(errs[0], P.CollectiveTimeoutError)
    assert errs[0].missing_ranks == (1,)
