"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):
    python tests/golden/gen_golden.py
It imports the reference from /root/reference/pkg/src (read-only, never
copied) and writes tests/golden/reference_golden.npz.  The GPU box has no
/root/reference; tests only read the committed .npz.

Cases (reference call sites in brackets):
  grid_*   : gradient-equivalence composition of cli.py:93-122 -- per-rank
             disco_step outputs via run_ranks (shard.py:169, fabric.py:291)
             and clip_grad_full (oracle.py:130) on seeded inputs
             (cli.py:103-105); B in {8,16,64}, D in {4,8,16}, N in {1,2,4,8},
             t in {1,10,100}, seed 0 (a slice of test_acceptance.py:31-58).
  flip_*   : same with flip_cross_rank_sign=True (test_acceptance.py:161-172).
  llg_*    : local_loss_and_grads contributions per rank (shard.py:98).
  readme   : the README library example B=32, D=8, N=4, t=100 (README.md:139-155).
  kat_*    : known answers (test_oracle.py:89-103, 131-138).
  cfgA     : config A of BASELINE.json -- B=1024, D=512, N=2, t=100, bf16-rounded
             features in f32 (the reference's bench precision, costs.py:158):
             loss, 32 sampled gradient rows, full-array sums.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import disco  # noqa: E402  (the reference package)
from disco import clip_grad_full, clip_loss_full, disco_step, l2_normalize_rows, run_ranks  # noqa: E402
from disco.shard import ShardLayout, local_loss_and_grads  # noqa: E402

from oracle.disco_oracle import bf16_round  # noqa: E402  (input rounding only)


def seeded(B, D, seed):
    rng = np.random.default_rng(seed)
    I = l2_normalize_rows(rng.standard_normal((B, D)))
    T = l2_normalize_rows(rng.standard_normal((B, D)))
    return I, T


def run_disco(I, T, world, t, **kw):
    b = I.shape[0] // world

    def fn(ep):
        rows = slice(ep.rank * b, (ep.rank + 1) * b)
        return disco_step(ep, I[rows], T[rows], t, **kw)

    res = run_ranks(world, fn)
    return (np.vstack([r[0] for r in res]), np.vstack([r[1] for r in res]),
            np.array([r[2] for r in res]))


def main():
    out = {}
    cases = []
    for B in (8, 16, 64):
        for D in (4, 8, 16):
            for N in (1, 2, 4, 8):
                if B % N:
                    continue
                for t in (1.0, 10.0, 100.0):
                    cases.append((B, D, N, t, 0))
    for i, (B, D, N, t, seed) in enumerate(cases):
        I, T = seeded(B, D, seed)
        di, dt, losses = run_disco(I, T, N, t)
        ref = clip_grad_full(I, T, t)
        key = f"grid_{i:03d}"
        out[key + "_meta"] = np.array([B, D, N, t, seed], dtype=np.float64)
        out[key + "_I"], out[key + "_T"] = I, T
        out[key + "_disco_image"], out[key + "_disco_text"], out[key + "_disco_loss"] = di, dt, losses
        out[key + "_oracle_image"], out[key + "_oracle_text"] = ref.d_image, ref.d_text
        out[key + "_oracle_loss"] = np.array([ref.loss.total, ref.loss.image_to_text, ref.loss.text_to_image])
    for i, (B, N) in enumerate(((8, 2), (16, 4), (64, 8))):
        I, T = seeded(B, 8, 0)
        di, dt, losses = run_disco(I, T, N, 10.0, flip_cross_rank_sign=True)
        out[f"flip_{i}_meta"] = np.array([B, 8, N, 10.0, 0])
        out[f"flip_{i}_image"], out[f"flip_{i}_text"], out[f"flip_{i}_loss"] = di, dt, losses
    # local_loss_and_grads contributions (test_shard.py:125-139 shape)
    rng = np.random.default_rng(3)
    m = rng.standard_normal((12, 5))
    I = m / np.linalg.norm(m, axis=1, keepdims=True)
    m = rng.standard_normal((12, 5))
    T = m / np.linalg.norm(m, axis=1, keepdims=True)
    out["llg_I"], out["llg_T"] = I, T
    for N in (2, 3, 4):
        for r in range(N):
            c = local_loss_and_grads(ShardLayout(world_size=N, global_batch=12, rank=r), I, T, 10.0)
            out[f"llg_{N}_{r}_image"], out[f"llg_{N}_{r}_text"] = c.d_image_full, c.d_text_full
            out[f"llg_{N}_{r}_loss"] = np.array([c.local_loss])
    # README example
    I, T = seeded(32, 8, 0)
    di, dt, losses = run_disco(I, T, 4, 100.0)
    out["readme_I"], out["readme_T"] = I, T
    out["readme_image"], out["readme_text"], out["readme_loss"] = di, dt, losses
    # known answers
    eye = np.eye(2)
    kl = clip_loss_full(eye, eye, 1.0)
    out["kat_eye_loss"] = np.array([kl.total, kl.image_to_text, kl.text_to_image])
    feats = np.tile(np.array([1.0, 0.0, 0.0]), (4, 1))
    out["kat_identical_loss"] = np.array([clip_loss_full(feats, feats, 10.0).total])
    one = clip_grad_full(np.array([[1.0, 0.0]]), np.array([[0.6, 0.8]]), 10.0)
    out["kat_single_loss"] = np.array([one.loss.total])
    out["kat_single_grad"] = np.concatenate([one.d_image, one.d_text])
    # config A, f32 bf16-rounded inputs (the reference's benchmark precision)
    I, T = seeded(1024, 512, 0)
    I32 = bf16_round(I)
    T32 = bf16_round(T)
    di, dt, losses = run_disco(I32, T32, 2, 100.0)
    ref = clip_grad_full(I32.astype(np.float64), T32.astype(np.float64), 100.0)
    rows = np.arange(0, 1024, 32)
    out["cfgA_rows"] = rows
    out["cfgA_disco_image_rows"], out["cfgA_disco_text_rows"] = di[rows], dt[rows]
    out["cfgA_disco_loss"] = losses
    out["cfgA_disco_sums"] = np.array([di.sum(), dt.sum(), np.abs(di).sum(), np.abs(dt).sum()])
    out["cfgA_oracle_image_rows"], out["cfgA_oracle_text_rows"] = ref.d_image[rows], ref.d_text[rows]
    out["cfgA_oracle_loss"] = np.array([ref.loss.total, ref.loss.image_to_text, ref.loss.text_to_image])
    out["cfgA_oracle_sums"] = np.array([ref.d_image.sum(), ref.d_text.sum(),
                                        np.abs(ref.d_image).sum(), np.abs(ref.d_text).sum()])
    out["reference_version"] = np.array([disco.__version__])
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(cases)} grid cases, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
