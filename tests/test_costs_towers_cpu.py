"""CPU: the cost model and the tower trainer's host logic against reference golden vectors.

tests/golden/reference_towers.npz comes from the unmodified reference
(tests/golden/gen_golden_towers.py).
"""

import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2304_08480_b200 import costs, towers
from paper_2304_08480_b200.errors import DomainError, LayoutError

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_towers.npz"))


def test_analytic_footprint_matches_reference_exactly():
    for row in G["analytic"]:
        mi, B, N, L, D, bps, backbone, loss_el, total, flops, nbytes = (int(v) for v in row)
        r = costs.analytic_footprint(costs.CostInputs(B=B, N=N, L=L, D=D, bytes_per_scalar=bps),
                                     costs.METHODS[mi])
        assert (r.backbone_elements, r.loss_elements, r.total_elements, r.loss_flops, r.bytes) == \
            (backbone, loss_el, total, flops, nbytes), (costs.METHODS[mi], B, N, L, D)


def test_savings_and_bytes_moved():
    assert costs.savings_fraction(1) == 0 and costs.savings_fraction(2) == 0
    assert costs.savings_fraction(8) == Fraction(3, 4)
    assert costs.bytes_moved("all_gather", 10, 4) == 40
    with pytest.raises(DomainError):
        costs.bytes_moved("broadcast", 1, 2)
    with pytest.raises(DomainError):
        costs.savings_fraction(0)


def test_cost_inputs_validation_and_formats():
    with pytest.raises(DomainError):
        costs.CostInputs(B=10, N=3, L=1, D=1, bytes_per_scalar=4)
    with pytest.raises(DomainError):
        costs.CostInputs(B=8, N=2, L=1, D=1, bytes_per_scalar=2)
    r = costs.analytic_footprint(costs.CostInputs(B=8, N=2, L=1, D=4, bytes_per_scalar=4), "DisCo")
    csv_text = costs.reports_to_csv([r])
    assert csv_text.splitlines()[0] == ",".join(costs.CSV_FIELDS)
    assert '"method": "DisCo"' in costs.reports_to_json([r])
    assert costs.reports_to_table([r]).splitlines()[0].split()[0] == "method"


def test_generate_dataset_and_weights_equal_reference_draws():
    ds = towers.generate_dataset(M=64, D_in=8, latent_dim=4, noise_scale=0.05, seed=0)
    assert np.array_equal(ds.image_inputs, G["ds_image"]) and np.array_equal(ds.text_inputs, G["ds_text"])
    W_i, W_t = towers.initial_weights(8, 4, seed=1)
    assert np.array_equal(W_i, G["W0_image"]) and np.array_equal(W_t, G["W0_text"])


def test_train_config_validation():
    with pytest.raises(LayoutError):
        towers.TrainConfig(global_batch=10, world_size=4, steps=1, learning_rate=0.1, seed=0, mode="disco")
    with pytest.raises(DomainError):
        towers.TrainConfig(global_batch=8, world_size=2, steps=1, learning_rate=0.1, seed=0, mode="other")
    with pytest.raises(DomainError):
        towers.generate_dataset(M=0, D_in=2, latent_dim=1, noise_scale=0.0, seed=0)
