"""Host-side API of the drop-in: names, validation order, exceptions (no device needed).

Mirrors the reference's own tests of the same entry points
(test_shard.py:30-97, 187-195, 269-274).
"""

import numpy as np
import pytest

import paper_2304_08480_b200 as P
from paper_2304_08480_b200 import DomainError, LayoutError, ShapeError, ShardLayout, local_labels, shard_slice


class TestShardLayout:
    def test_slice_and_local_batch(self):
        layout = ShardLayout(world_size=2, global_batch=8, rank=1)
        assert layout.local_batch == 4
        assert layout.row_slice == slice(4, 8)

    def test_divisibility_error_names_both_values(self):
        with pytest.raises(LayoutError, match=r"8.*3|3.*8"):
            ShardLayout(world_size=3, global_batch=8, rank=0)

    def test_bounds(self):
        for kw in (dict(world_size=0, global_batch=4, rank=0), dict(world_size=2, global_batch=0, rank=0),
                   dict(world_size=2, global_batch=4, rank=2), dict(world_size=2, global_batch=4, rank=-1)):
            with pytest.raises(LayoutError):
                ShardLayout(**kw)


def test_shard_slice_and_labels():
    full = np.arange(8.0).reshape(4, 2)
    layout = ShardLayout(world_size=2, global_batch=4, rank=1)
    block = shard_slice(layout, full)
    assert np.shares_memory(block, full) and block.tolist() == [[4.0, 5.0], [6.0, 7.0]]
    with pytest.raises(LayoutError):
        shard_slice(layout, np.zeros((6, 2)))
    assert local_labels(ShardLayout(world_size=3, global_batch=12, rank=2)).tolist() == [8, 9, 10, 11]


def test_local_loss_and_grads_validation_order():
    # shard.py:112-120: DomainError, then ShapeError, then LayoutError -- all before any device work
    layout = ShardLayout(world_size=2, global_batch=4, rank=0)
    good = np.eye(4)
    with pytest.raises(DomainError):
        P.local_loss_and_grads(layout, good, good, 0.0)
    with pytest.raises(ShapeError):
        P.local_loss_and_grads(layout, good, np.eye(4)[:, :3], 1.0)
    with pytest.raises(LayoutError):
        P.local_loss_and_grads(layout, np.eye(6), np.eye(6), 1.0)


def test_disco_step_validation():
    class Ep:
        rank, world_size = 0, 2
    with pytest.raises(ShapeError):
        P.disco_step(Ep(), np.eye(2), np.eye(3)[:2], 1.0)
    with pytest.raises(DomainError):
        P.disco_step(Ep(), np.eye(2), np.eye(2), -1.0)

    class Bad:
        rank, world_size = 2, 2
    with pytest.raises(LayoutError):
        P.disco_step(Bad(), np.eye(2), np.eye(2), 1.0)


def test_reference_names_are_exported():
    # the names of reference __init__.py:53-60 that belong to the hot path
    for name in ("disco_step", "local_loss_and_grads", "ShardLayout", "LocalGradContribution", "local_labels",
                 "shard_slice", "ReduceOp", "run_ranks", "Counters", "tracking", "ShapeError", "LayoutError",
                 "DomainError", "CollectiveContractError", "CollectiveTimeoutError", "DeadlockError"):
        assert hasattr(P, name), name


def test_counters_match_reference_accounting():
    from paper_2304_08480_b200.shard import _account_loss_scope
    loss, exch = P.Counters(), P.Counters()
    b, B, D = 4, 8, 4
    _account_loss_scope(loss, exch, b, B, D)
    # test_shard.py:181-185
    assert loss.peak_live_elements == 2 * b * B and loss.live_elements == 0
    assert loss.flops == 4 * b * B * D
    assert exch.peak_live_elements == 2 * B * D and exch.flops == 8 * b * B * D


def test_row_blocks_partition_rows():
    """The pipelined read-back's row blocks partition [0, b) into non-empty, 256-aligned blocks."""
    from paper_2304_08480_b200.shard import row_blocks
    for b in (256, 1792, 2048, 2304, 3072, 4096, 8192, 32768, 65536, 196608 // 8):
        bl = row_blocks(b)
        assert bl[0][0] == 0 and bl[-1][1] == b
        assert all(hi > lo for lo, hi in bl)
        assert all(bl[i][1] == bl[i + 1][0] for i in range(len(bl) - 1))
        assert all(lo % 256 == 0 for lo, _ in bl)


def test_fused_row_blocks_whole_waves():
    """Fused single-rank backward row blocks: one wave of 74 CTA pairs (4 units per 256-row tile)
    each; a partition of [0, b) on 256-row boundaries."""
    from paper_2304_08480_b200.shard import fused_row_blocks
    bl = fused_row_blocks(32768, 74)
    assert [(hi - lo) // 256 for lo, hi in bl] == [18] * 7 + [2]
    for b in (4096, 8192, 16384, 32768, 65536, 12288):
        bl = fused_row_blocks(b, 74)
        assert bl[0][0] == 0 and bl[-1][1] == b
        assert all(lo < hi and lo % 256 == 0 for lo, hi in bl)
        assert all(bl[i][1] == bl[i + 1][0] for i in range(len(bl) - 1))
