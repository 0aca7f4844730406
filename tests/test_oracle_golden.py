"""Pin the CPU oracle (oracle/disco_oracle.py) to outputs of the reference itself.

tests/golden/reference_golden.npz was produced by tests/golden/gen_golden.py
running the unmodified reference package.  Tolerance 1e-12 as in the
reference's acceptance grid (test_acceptance.py:51).
"""

import math
import os

import numpy as np
import pytest

from oracle import disco_oracle as O

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))
GRID = sorted({k[:8] for k in GOLD.files if k.startswith("grid_")})


@pytest.mark.parametrize("key", GRID)
def test_grid_case_matches_reference(key):
    B, D, N, t, seed = GOLD[key + "_meta"]
    B, D, N = int(B), int(D), int(N)
    I, T = GOLD[key + "_I"], GOLD[key + "_T"]
    # inputs regenerate bit-exactly from the seed (cli.py:103-105)
    rI, rT = O.synthetic_features(B, D, int(seed), bf16=False)
    assert rI.tobytes() == I.tobytes() and rT.tobytes() == T.tobytes()
    oi, ot, (total, i2t, t2i) = O.clip_grad_full(I, T, t)
    assert O.max_rel_error(oi, GOLD[key + "_oracle_image"]) < 1e-12
    assert O.max_rel_error(ot, GOLD[key + "_oracle_text"]) < 1e-12
    assert abs(total - GOLD[key + "_oracle_loss"][0]) < 1e-12
    assert abs(i2t - GOLD[key + "_oracle_loss"][1]) < 1e-12
    di, dt, loss = O.disco_step_all(I, T, N, t)
    assert O.max_rel_error(di, GOLD[key + "_disco_image"]) < 1e-12
    assert O.max_rel_error(dt, GOLD[key + "_disco_text"]) < 1e-12
    assert np.all(np.abs(GOLD[key + "_disco_loss"] - loss) < 1e-12)


@pytest.mark.parametrize("i", range(3))
def test_flip_hook_matches_reference(i):
    B, D, N, t, seed = GOLD[f"flip_{i}_meta"]
    I, T = O.synthetic_features(int(B), int(D), int(seed), bf16=False)
    di, dt, loss = O.disco_step_all(I, T, int(N), t, flip_cross_rank_sign=True)
    assert O.max_rel_error(di, GOLD[f"flip_{i}_image"]) < 1e-12
    assert O.max_rel_error(dt, GOLD[f"flip_{i}_text"]) < 1e-12
    ref_i, _, _ = O.clip_grad_full(I, T, t)
    assert O.max_rel_error(di, ref_i) > 1e-3  # the mutation is visible


@pytest.mark.parametrize("N", [2, 3, 4])
def test_local_contributions_match_reference(N):
    I, T = GOLD["llg_I"], GOLD["llg_T"]
    for r in range(N):
        di, dt, loss = O.local_loss_and_grads(N, r, I, T, 10.0)
        assert O.max_rel_error(di, GOLD[f"llg_{N}_{r}_image"]) < 1e-12
        assert O.max_rel_error(dt, GOLD[f"llg_{N}_{r}_text"]) < 1e-12
        assert abs(loss - GOLD[f"llg_{N}_{r}_loss"][0]) < 1e-12


def test_readme_example():
    I, T = GOLD["readme_I"], GOLD["readme_T"]
    di, dt, loss = O.disco_step_all(I, T, 4, 100.0)
    assert O.max_rel_error(di, GOLD["readme_image"]) < 1e-12
    assert O.max_rel_error(dt, GOLD["readme_text"]) < 1e-12
    ref_i, _, _ = O.clip_grad_full(I, T, 100.0)
    assert np.max(np.abs(di - ref_i)) < 1e-12


def test_known_answers():
    expected = math.log(1.0 + math.exp(-1.0))  # test_oracle.py:89-97
    total, i2t, t2i = O.clip_loss_full(np.eye(2), np.eye(2), 1.0)
    assert abs(total - expected) < 1e-14 and abs(i2t - expected) < 1e-14
    assert np.allclose(GOLD["kat_eye_loss"], expected, atol=1e-14)
    feats = np.tile(np.array([1.0, 0.0, 0.0]), (4, 1))
    assert abs(O.clip_loss_full(feats, feats, 10.0)[0] - math.log(4.0)) < 1e-14
    assert abs(GOLD["kat_identical_loss"][0] - math.log(4.0)) < 1e-14
    di, dt, loss = O.clip_grad_full(np.array([[1.0, 0.0]]), np.array([[0.6, 0.8]]), 10.0)
    assert loss[0] == 0.0 and not di.any() and not dt.any()
    assert GOLD["kat_single_loss"][0] == 0.0 and not GOLD["kat_single_grad"].any()


def test_config_a_matches_reference():
    I, T = O.synthetic_features(1024, 512, 0)   # bf16-rounded, f64 carrier
    rows = GOLD["cfgA_rows"]
    oi, ot, loss = O.clip_grad_full(I, T, 100.0)
    assert O.max_rel_error(oi[rows], GOLD["cfgA_oracle_image_rows"]) < 1e-12
    assert O.max_rel_error(ot[rows], GOLD["cfgA_oracle_text_rows"]) < 1e-12
    assert abs(loss[0] - GOLD["cfgA_oracle_loss"][0]) < 1e-12
    sums = np.array([oi.sum(), ot.sum(), np.abs(oi).sum(), np.abs(ot).sum()])
    assert np.allclose(sums, GOLD["cfgA_oracle_sums"], rtol=1e-10, atol=1e-12)
    # the reference's f32 disco path agrees with the f64 oracle to f32 rounding
    assert O.max_rel_error(GOLD["cfgA_disco_image_rows"], GOLD["cfgA_oracle_image_rows"]) < 1e-5
    # the blocked/sampled-row oracle used at B=32K agrees with the dense one
    ri, rt, rloss = O.clip_grad_rows(I, T, 100.0, rows)
    assert O.max_rel_error(ri, oi[rows]) < 1e-12
    assert O.max_rel_error(rt, ot[rows]) < 1e-12
    assert abs(rloss[0] - loss[0]) < 1e-12


def test_bf16_round_is_round_to_nearest_even():
    import torch
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32)
    ours = O.bf16_round(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert ours.tobytes() == ref.tobytes()


@pytest.mark.parametrize("t", [1.0, 14.2857, 100.0])
@pytest.mark.parametrize("correlated", [False, True])
def test_dlogit_scale_oracle_matches_finite_difference(t, correlated):
    """oracle.dlogit_scale_full (the logit-scale gradient the reference lacks)
    against a central difference of the reference-pinned clip_loss_full."""
    I, T = O.synthetic_features(64, 16, 7, correlated=correlated, bf16=False)
    h = 1e-5 * t
    fd = (O.clip_loss_full(I, T, t + h)[0] - O.clip_loss_full(I, T, t - h)[0]) / (2 * h)
    g = O.dlogit_scale_full(I, T, t)
    assert abs(g - fd) <= 1e-6 * max(1.0, abs(fd)), (g, fd)


def test_dlogit_scale_euler_identity():
    """dL/dt = (<dL/dI, I> + <dL/dT, T>) / (2t) (the identity the device path uses)."""
    I, T = O.synthetic_features(48, 8, 2, bf16=False)
    t = 10.0
    di, dt, _ = O.clip_grad_full(I, T, t)
    assert abs(O.dlogit_scale_full(I, T, t) - ((di * I).sum() + (dt * T).sum()) / (2 * t)) < 1e-12


@pytest.mark.parametrize("world", [1, 2, 4])
def test_blocked_timing_port_equals_the_oracle_step(world):
    """oracle.disco_step_blocked (the CPU baseline's timing kernel) computes the same step as
    disco_step_all (itself pinned to the reference above), for any blocking and thread count."""
    I, T = O.synthetic_features(64, 8, 3)
    ref = O.disco_step_all(I, T, world, 10.0)
    for rows, workers in ((5, 3), (64, 1), (7, 8)):
        got = O.disco_step_blocked(I, T, world, 10.0, rows_per_block=rows, workers=workers)
        assert O.max_rel_error(got[0], ref[0]) < 1e-12
        assert O.max_rel_error(got[1], ref[1]) < 1e-12
        assert abs(got[2] - ref[2]) < 1e-12 * abs(ref[2])
