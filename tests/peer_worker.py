"""One rank of the two-process tests in tests/test_gpu_peer.py (not collected by pytest).

Both ranks share cuda:0; the process group is gloo.  argv[2] selects the exchange:
  peer  -- the gradient exchange is the peer transport over CUDA IPC-mapped windows;
  nccl  -- DISCO_PEER=0: the exchange the NCCL path runs (ProcessGroupEndpoint.all_gather_into,
           all_to_all_into, the per-row ce all_gather) with the real device kernels, the
           collectives staged through host memory (gloo cannot move CUDA tensors; two ranks on
           one GPU cannot form an NCCL communicator);
  fallback -- the peer transport is requested but reported unavailable (peer access check patched
           to fail): every rank must fall back to the NCCL exchange together.
Two steps, so both parity windows are used.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_08480_b200 as P  # noqa: E402


def main(out_dir, mode="peer"):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if mode == "fallback":
        from paper_2304_08480_b200 import peer as peer_mod
        peer_mod._peer_access_all_pairs = lambda devices: False
    ep = P.ProcessGroupEndpoint(peer=(mode != "nccl"))
    I = np.load(os.path.join(out_dir, "I.npy"))
    T = np.load(os.path.join(out_dir, "T.npy"))
    b = I.shape[0] // world
    Id = torch.from_numpy(I[rank * b:(rank + 1) * b]).cuda()
    Td = torch.from_numpy(T[rank * b:(rank + 1) * b]).cuda()
    for _ in range(2):
        di, dt, loss = P.disco_step(ep, Id, Td, 100.0)
    if mode == "fallback":
        assert ep.peer is False, "peer transport should have been disabled"
    np.save(os.path.join(out_dir, f"di{rank}.npy"), di.cpu().numpy())
    np.save(os.path.join(out_dir, f"dt{rank}.npy"), dt.cpu().numpy())
    np.save(os.path.join(out_dir, f"loss{rank}.npy"), np.array(loss))
    ep.barrier()
    from paper_2304_08480_b200.shard import clear_plans
    clear_plans()
    ep.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "peer")
