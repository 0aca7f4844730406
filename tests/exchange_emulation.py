"""Test-only numpy emulation of the device dataflow's REDUCTION ORDER.

It mirrors, in f32 numpy, the order in which paper_2304_08480_b200's kernels
combine partial results, so the N-invariance argument can be checked on a CPU
with real collectives (gloo) and compared with the CPU oracle:

  canonical chunks  : 8 when B % 1024 == 0 and N | 8, else N   (disco_b200_chunking)
  cross partials    : one per canonical row chunk, X_k = G[chunk rows]^T A[chunk rows]
  pair level        : (X_2i + X_2i+1) in the GEMM epilogue
  sender presum     : balanced tree over the rank's pair partials -> destination-major slabs
  exchange          : all_to_all of [N][2][b][D] slabs
  owner combine     : balanced tree over sources (power-of-two N), ascending otherwise,
                      then s * (intra + cross), s = 0.5 t / B
  loss              : per-row ce gathered, summed in global-row order

Row-local quantities (softmax rows, intra products) are computed per fixed
128-row block so they do not depend on how many rows a rank holds.
"""

import numpy as np


def chunking(B, N):
    if B % 1024 == 0 and 8 % N == 0:
        return 8, 8 // N
    return N, 1


def tree(xs):
    n = len(xs)
    if n & (n - 1) == 0 and n <= 8:
        xs = list(xs)
        w = 1
        while w < n:
            for k in range(0, n - w, 2 * w):
                xs[k] = xs[k] + xs[k + w]
            w *= 2
        return xs[0]
    acc = xs[0]
    for x in xs[1:]:
        acc = acc + x
    return acc


def rows_blockwise(fn, n_rows, block=128):
    return np.concatenate([fn(slice(s, min(s + block, n_rows))) for s in range(0, n_rows, block)], axis=0)


def local_phase(rank, N, I, T, t, leaves=False):
    """Everything before the exchange on one rank: G blocks, intra terms, slabs, per-row ce.

    leaves=True (peer transport): instead of the presummed slabs, return the rank's chunk
    partials (pair level applied) as [np][2][B][D] -- what the GEMM pushes to the owners."""
    B, D = I.shape
    b = B // N
    nch, cpr = chunking(B, N)
    Bc = B // nch
    lo = rank * b
    t32 = np.float32(t)
    feats = (I.astype(np.float32), T.astype(np.float32))
    G, ce = [], []
    for d in range(2):
        A, C = feats[d], feats[1 - d]

        def g_rows(sl):
            S = (A[lo + sl.start:lo + sl.stop] @ C.T) * t32
            m = S.max(axis=1, keepdims=True)
            P = np.exp(S - m)
            P /= P.sum(axis=1, keepdims=True)
            lab = np.arange(sl.start, sl.stop) + lo
            out = P.copy()
            out[np.arange(len(lab)), lab] -= 1.0
            return out

        G.append(rows_blockwise(g_rows, b).astype(np.float32))
        S_loc = (A[lo:lo + b] @ C.T).astype(np.float64) * t
        lab = np.arange(b) + lo
        mx = S_loc.max(axis=1)
        ce.append(np.log(np.exp(S_loc - mx[:, None]).sum(axis=1)) + mx - S_loc[np.arange(b), lab])
    # gradient index g: image (0) <- intra G_i.T_g, cross G_t^T.T_n ; text (1) <- G_t.I_g, G_i^T.I_n
    intra = [rows_blockwise(lambda sl: G[0][sl] @ feats[1], b), rows_blockwise(lambda sl: G[1][sl] @ feats[0], b)]
    slabs, leaf_parts = [], []
    for g in range(2):
        Gd, Ad = (G[1], feats[1]) if g == 0 else (G[0], feats[0])
        parts = []
        for j in range(cpr):
            r0 = j * (Bc if cpr > 1 else b)
            r1 = r0 + (Bc if cpr > 1 else b)
            parts.append(Gd[r0:r1].T @ Ad[lo + r0:lo + r1])     # B x D, one canonical chunk
        if cpr >= 2:
            parts = [parts[2 * i] + parts[2 * i + 1] for i in range(cpr // 2)]
        leaf_parts.append(parts)
        slabs.append(tree(parts))
    if leaves:
        lv = np.stack([np.stack([leaf_parts[g][k] for g in range(2)]) for k in range(len(leaf_parts[0]))])
        return np.stack(intra), lv.astype(np.float32), np.stack(ce).astype(np.float32)
    send = np.stack([np.stack([slabs[g][dst * b:(dst + 1) * b] for g in range(2)]) for dst in range(N)])
    return np.stack(intra), send.astype(np.float32), np.stack(ce).astype(np.float32)


def owner_phase(rank, N, t, B, intra, recv):
    """After the exchange: s * (intra + tree over sources of the received slabs)."""
    s = np.float32(0.5 * t / B)
    cross = [tree([recv[src][g] for src in range(N)]) for g in range(2)]
    return [(intra[g] + cross[g]) * s for g in range(2)]


def loss_from(ce_all, N, b):
    """ce_all: [N][2][b] -> f64 sum in (dir, global row) order / 2B."""
    B = N * b
    flat = np.concatenate([ce_all[:, d, :].reshape(-1) for d in range(2)]).astype(np.float64)
    return float(np.sum(flat) / (2 * B))


def run_single_process(N, I, T, t):
    """All ranks in one process, exchange by array transposition."""
    B = I.shape[0]
    b = B // N
    outs = [local_phase(r, N, I, T, t) for r in range(N)]
    grads = []
    for r in range(N):
        recv = np.stack([outs[src][1][r] for src in range(N)])
        grads.append(owner_phase(r, N, t, B, outs[r][0], recv))
    d_image = np.concatenate([g[0] for g in grads])
    d_text = np.concatenate([g[1] for g in grads])
    loss = loss_from(np.stack([o[2] for o in outs]), N, b)
    return d_image, d_text, loss


def run_single_process_peer(N, I, T, t):
    """Peer transport: every rank pushes its leaves (no sender presum) into the owners' windows
    [2][L][b][D] (leaf src*np + k); the owner's tree runs over all L = N*np leaves."""
    B = I.shape[0]
    b = B // N
    outs = [local_phase(r, N, I, T, t, leaves=True) for r in range(N)]
    s = np.float32(0.5 * t / B)
    grads = []
    for r in range(N):
        window = [[outs[src][1][k][g][r * b:(r + 1) * b] for src in range(N) for k in range(outs[src][1].shape[0])]
                  for g in range(2)]
        grads.append([(outs[r][0][g] + tree(window[g])) * s for g in range(2)])
    d_image = np.concatenate([g[0] for g in grads])
    d_text = np.concatenate([g[1] for g in grads])
    loss = loss_from(np.stack([o[2] for o in outs]), N, b)
    return d_image, d_text, loss
