"""CPU oracle for the DisCo loss path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only tests/, the smoke()
entry of __graft_entry__.py and bench.py's ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The shipped package (paper_2304_08480_b200)
never imports it and has no CPU fallback.

It is a numpy restatement of the reference package's algorithm
(/root/reference/pkg/src/disco, numpy>=1.24, pyproject.toml:10), each
function citing the reference lines it follows.  Row loops of the reference
are vectorised (identical arithmetic per row, f64 by default).  Parity of
this restatement is pinned against outputs of the reference itself:
tests/golden/gen_golden.py imports the reference in the build container and
stores them in tests/golden/*.npz; tests/test_oracle_golden.py checks this
module against them at 1e-12 (the reference's own tolerance,
test_acceptance.py:51).
"""

from __future__ import annotations

import math

import numpy as np

NORM_EPSILON = 1e-12  # matrix.py:24


# ---------------------------------------------------------------------------
# dense helpers (matrix.py)
# ---------------------------------------------------------------------------
def l2_normalize_rows(m: np.ndarray) -> np.ndarray:
    """matrix.py:165-176: scale each row to unit Euclidean norm."""
    norms = np.linalg.norm(m, axis=1, keepdims=True)
    if norms.min() < NORM_EPSILON:
        raise ValueError("row norm below epsilon")
    return m / norms


def max_rel_error(actual, expected) -> float:
    """matrix.py:147-162: max |a - e| / max |e| (normwise); 0/0 -> 0, x/0 -> inf."""
    actual = np.asarray(actual, dtype=np.float64)
    expected = np.asarray(expected, dtype=np.float64)
    if actual.shape != expected.shape:
        raise ValueError(f"shapes disagree: {actual.shape} vs {expected.shape}")
    diff = float(np.abs(actual - expected).max()) if actual.size else 0.0
    scale = float(np.abs(expected).max()) if expected.size else 0.0
    if scale == 0.0:
        return 0.0 if diff == 0.0 else float("inf")
    return diff / scale


def row_ce(logits: np.ndarray, labels: np.ndarray) -> np.ndarray:
    """Per-row terms of matrix.py:103-118: m + log(sum exp(row - m)) - row[label]."""
    m = logits.max(axis=1)
    lse = np.log(np.exp(logits - m[:, None]).sum(axis=1)) + m
    return lse - logits[np.arange(logits.shape[0]), labels]


def cross_entropy_mean(logits: np.ndarray, labels) -> float:
    """matrix.py:103-118 (mean over rows, f64 accumulation)."""
    labels = np.asarray(labels)
    return float(row_ce(logits, labels).sum() / logits.shape[0])


def softmax_ce_grad_inplace(m: np.ndarray, labels: np.ndarray, scale: float) -> None:
    """matrix.py:131-144: m <- scale * (row_softmax(m) - onehot(labels))."""
    m -= m.max(axis=1, keepdims=True)
    np.exp(m, out=m)
    m /= m.sum(axis=1, keepdims=True)
    m[np.arange(m.shape[0]), labels] -= 1.0
    m *= scale


# ---------------------------------------------------------------------------
# full-batch oracle (oracle.py)
# ---------------------------------------------------------------------------
def clip_loss_full(I, T, t: float):
    """oracle.py:108-127 -> (total, image_to_text, text_to_image)."""
    I = np.asarray(I)
    T = np.asarray(T)
    S = (I @ T.T) * t
    labels = np.arange(I.shape[0])
    i2t = cross_entropy_mean(S, labels)
    t2i = cross_entropy_mean(np.ascontiguousarray(S.T), labels)
    return (i2t + t2i) / 2.0, i2t, t2i


def clip_grad_full(I, T, t: float):
    """oracle.py:130-200 -> (d_image, d_text, (total, i2t, t2i)).

    Row and column softmax statistics of S = t*I@T.T, then
    G = (P1 - Y + (P2 - Y).T) / (2B), d_image = t*G@T, d_text = t*G.T@I.
    """
    I = np.asarray(I, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    B = I.shape[0]
    S = I @ T.T
    S *= t
    diag = S.diagonal().copy()
    row_max = S.max(axis=1)
    row_sum = np.exp(S - row_max[:, None]).sum(axis=1)
    col_max = S.max(axis=0)
    col_sum = np.exp(S - col_max[None, :]).sum(axis=0)
    i2t = float(np.mean(np.log(row_sum) + row_max - diag))
    t2i = float(np.mean(np.log(col_sum) + col_max - diag))
    col_part = np.exp(S - col_max[None, :]) / col_sum[None, :]
    S -= row_max[:, None]
    np.exp(S, out=S)
    S /= row_sum[:, None]
    S += col_part
    del col_part
    S[np.arange(B), np.arange(B)] -= 2.0
    S *= 1.0 / (2.0 * B)
    d_image = (S @ T) * t
    d_text = (S.T @ I) * t
    return d_image, d_text, ((i2t + t2i) / 2.0, i2t, t2i)


def dlogit_scale_full(I, T, t: float) -> float:
    """dL/dt of clip_loss_full (oracle.py:108-127) w.r.t. the logit scale t, f64.

    The reference computes no logit-scale gradient (a documented gap,
    SPEC.md:243), so this is pinned by finite differences of clip_loss_full
    (tests/test_oracle_golden.py), not by reference outputs.  With S = t*I@T.T
    and G = dL/dS = (P_row - Y + P_col - Y) / (2B) (oracle.py:130-200):
    dL/dt = sum(G * I@T.T).
    """
    I = np.asarray(I, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    B = I.shape[0]
    S0 = I @ T.T
    S = S0 * t
    P1 = np.exp(S - S.max(axis=1, keepdims=True))
    P1 /= P1.sum(axis=1, keepdims=True)
    P2 = np.exp(S - S.max(axis=0, keepdims=True))
    P2 /= P2.sum(axis=0, keepdims=True)
    G = P1 + P2
    G[np.arange(B), np.arange(B)] -= 2.0
    return float((G * S0).sum() / (2.0 * B))


def clip_stats_blocked(I, T, t: float, block: int = 2048):
    """Row/column softmax statistics of S = t*I@T.T without materialising S.

    Same quantities as oracle.py:157-171, streamed over row blocks so the
    B=32K parity checks fit in host memory.  Returns
    (row_max, row_sum, col_max, col_sum, diag, loss_tuple).
    """
    I = np.asarray(I, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    B = I.shape[0]
    row_max = np.empty(B)
    row_sum = np.empty(B)
    col_max = np.full(B, -np.inf)
    col_sum = np.zeros(B)
    diag = np.einsum("ij,ij->i", I, T) * t
    for s in range(0, B, block):
        blk = (I[s:s + block] @ T.T) * t
        rm = blk.max(axis=1)
        row_max[s:s + block] = rm
        row_sum[s:s + block] = np.exp(blk - rm[:, None]).sum(axis=1)
        cm = np.maximum(col_max, blk.max(axis=0))
        col_sum = col_sum * np.exp(col_max - cm) + np.exp(blk - cm[None, :]).sum(axis=0)
        col_max = cm
    i2t = float(np.mean(np.log(row_sum) + row_max - diag))
    t2i = float(np.mean(np.log(col_sum) + col_max - diag))
    return row_max, row_sum, col_max, col_sum, diag, ((i2t + t2i) / 2.0, i2t, t2i)


def clip_grad_rows(I, T, t: float, rows, stats=None):
    """Selected rows of clip_grad_full's d_image and d_text (oracle.py:173-191).

    Row j of d_image needs row j of G (row j of S plus column stats); row j of
    d_text needs column j of G (column j of S plus row stats).
    """
    I = np.asarray(I, dtype=np.float64)
    T = np.asarray(T, dtype=np.float64)
    B = I.shape[0]
    rows = np.asarray(rows)
    if stats is None:
        stats = clip_stats_blocked(I, T, t)
    row_max, row_sum, col_max, col_sum, _, loss = stats
    Srow = (I[rows] @ T.T) * t                   # S[j, :]
    Grow = np.exp(Srow - row_max[rows, None]) / row_sum[rows, None] \
        + np.exp(Srow - col_max[None, :]) / col_sum[None, :]
    Grow[np.arange(len(rows)), rows] -= 2.0
    Grow /= 2.0 * B
    Scol = (I @ T[rows].T).T * t                 # S[:, j] as rows
    Gcol = np.exp(Scol - row_max[None, :]) / row_sum[None, :] \
        + np.exp(Scol - col_max[rows, None]) / col_sum[rows, None]
    Gcol[np.arange(len(rows)), rows] -= 2.0
    Gcol /= 2.0 * B
    return (Grow @ T) * t, (Gcol @ I) * t, loss


# ---------------------------------------------------------------------------
# sharded path (shard.py + fabric.py semantics)
# ---------------------------------------------------------------------------
def local_loss_and_grads(world: int, rank: int, I_g, T_g, t: float, flip_cross_rank_sign: bool = False):
    """shard.py:98-166 -> (d_image_full, d_text_full, local_loss)."""
    I_g = np.asarray(I_g)
    T_g = np.asarray(T_g)
    B, _ = I_g.shape
    b = B // world
    rows = slice(rank * b, (rank + 1) * b)
    I_n, T_n = I_g[rows], T_g[rows]
    labels = np.arange(b) + b * rank
    logits_i = (I_n @ T_g.T) * t
    logits_t = (T_n @ I_g.T) * t
    local_loss = (cross_entropy_mean(logits_i, labels) + cross_entropy_mean(logits_t, labels)) / 2.0
    softmax_ce_grad_inplace(logits_i, labels, 0.5 / b)
    softmax_ce_grad_inplace(logits_t, labels, 0.5 / b)
    d_image = logits_t.T @ T_n
    d_image[rows] += logits_i @ T_g
    d_text = logits_i.T @ I_n
    d_text[rows] += logits_t @ I_g
    d_image *= t
    d_text *= t
    if flip_cross_rank_sign:
        for d in (d_image, d_text):
            d[:rows.start] *= -1.0
            d[rows.stop:] *= -1.0
    return d_image, d_text, float(local_loss)


def disco_step_all(I, T, world: int, t: float, flip_cross_rank_sign: bool = False):
    """All ranks of shard.py:169-208 with fabric.py:81-100 reductions.

    all_reduce(AVG) = ascending-rank sum then one division; the scalar loss
    likewise.  Returns the row-stacked per-rank slices and the global loss.
    """
    I = np.asarray(I)
    T = np.asarray(T)
    parts = [local_loss_and_grads(world, r, I, T, t, flip_cross_rank_sign) for r in range(world)]
    acc_i = parts[0][0].copy()
    acc_t = parts[0][1].copy()
    loss = float(parts[0][2])
    for p in parts[1:]:
        acc_i += p[0]
        acc_t += p[1]
        loss += p[2]
    acc_i /= world
    acc_t /= world
    loss /= world
    return acc_i, acc_t, loss


def disco_step_blocked(I, T, world: int, t: float, rows_per_block: int = 1024, workers: int = 1):
    """All ranks of shard.py:169-208 computed in row blocks on a thread pool: the CPU baseline's
    timing kernel (bench.py ``--impl reference`` / ``cpu_baseline``), NOT a parity oracle.

    Same arithmetic as ``disco_step_all`` in the dtype of the inputs (f32 in the bench, the
    reference's benchmark precision, costs.py:158): for rank n and each block of its rows
    (labels n*b + arange, shard.py:92-95), logits = t * rows @ gathered.T (shard.py:134-137),
    row CE (matrix.py:103-118), G = (softmax - onehot) * 0.5/b in place (matrix.py:131-144),
    then the cross terms G^T @ rows accumulated into full-size B x D contributions and the
    intra terms G @ gathered written into the block's rows (shard.py:148-154); the contributions
    are averaged over ranks (fabric.py:86-93) and the loss likewise.  The blocks of one rank's
    step are independent except for the cross accumulation, which each worker keeps in its own
    buffer and which is summed in worker order at the end.  numpy releases the GIL in BLAS and
    large ufuncs, so ``workers`` threads each run single-threaded BLAS on their own blocks.
    Returns (d_image, d_text, loss) for all B rows.
    """
    from concurrent.futures import ThreadPoolExecutor

    I = np.ascontiguousarray(I)
    T = np.ascontiguousarray(T)
    B, D = I.shape
    b = B // world
    dt = I.dtype.type
    tasks = []
    for n in range(world):
        for r0 in range(n * b, (n + 1) * b, rows_per_block):
            tasks.append((n, r0, min(r0 + rows_per_block, (n + 1) * b)))
    workers = max(1, min(workers, len(tasks)))
    parts = [tasks[w::workers] for w in range(workers)]
    intra_i = np.zeros((B, D), dtype=I.dtype)
    intra_t = np.zeros((B, D), dtype=I.dtype)

    def run(mine):
        cross_i = np.zeros((B, D), dtype=I.dtype)
        cross_t = np.zeros((B, D), dtype=I.dtype)
        ce = 0.0
        for n, r0, r1 in mine:
            labels = np.arange(r0, r1)
            li = (I[r0:r1] @ T.T) * dt(t)
            lt = (T[r0:r1] @ I.T) * dt(t)
            ce += float(row_ce(li, labels).sum() + row_ce(lt, labels).sum())
            softmax_ce_grad_inplace(li, labels, 0.5 / b)
            softmax_ce_grad_inplace(lt, labels, 0.5 / b)
            cross_i += lt.T @ T[r0:r1]
            cross_t += li.T @ I[r0:r1]
            intra_i[r0:r1] = li @ T
            intra_t[r0:r1] = lt @ I
        return cross_i, cross_t, ce

    if workers == 1:
        results = [run(parts[0])]
    else:
        with ThreadPoolExecutor(workers) as pool:
            results = list(pool.map(run, parts))
    d_image = intra_i
    d_text = intra_t
    ce = 0.0
    for ci, ct, c in results:
        d_image += ci
        d_text += ct
        ce += c
    d_image *= dt(t / world)
    d_text *= dt(t / world)
    loss = ce / (2.0 * b) / world
    return d_image, d_text, loss


# ---------------------------------------------------------------------------
# inputs and the parity metric composition (cli.py)
# ---------------------------------------------------------------------------
def bf16_round(x) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32 (exact values)."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def synthetic_features(B: int, D: int, seed: int, correlated: bool = False, bf16: bool = True):
    """cli.py:103-105: I then T from default_rng(seed), rows L2-normalised.

    ``correlated`` gives T = normalize(I + 3 g / sqrt(D)) (peaked softmax).
    Returns f64 arrays holding bf16-representable values when ``bf16``.
    """
    rng = np.random.default_rng(seed)
    I = l2_normalize_rows(rng.standard_normal((B, D)))
    g = rng.standard_normal((B, D))
    T = l2_normalize_rows(I + 3.0 * g / math.sqrt(D)) if correlated else l2_normalize_rows(g)
    if bf16:
        I = bf16_round(I).astype(np.float64)
        T = bf16_round(T).astype(np.float64)
    return I, T


def gradient_equivalence_error(d_image, d_text, loss, I, T, t: float) -> float:
    """cli.py:114-122: max of the three normwise errors against clip_grad_full."""
    ref_i, ref_t, ref_loss = clip_grad_full(I, T, t)
    return max(max_rel_error(d_image, ref_i), max_rel_error(d_text, ref_t),
               max_rel_error(np.array([loss]), np.array([ref_loss[0]])))
