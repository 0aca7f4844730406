"""The C-ABI library loads on a CPU-only host and exports every symbol of include/disco_b200.h.

Only host-side entry points (geometry, workspace layout, chunking) are called
here; nothing touches a device.
"""

import ctypes
import os
import re

import pytest

from paper_2304_08480_b200 import _lib
from paper_2304_08480_b200.errors import LayoutError, ShapeError

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "disco_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(disco_b200_\w+)\s*\(", text)))


def test_library_builds_and_loads():
    from paper_2304_08480_b200 import build
    build.build()
    lib = _lib.load()
    assert lib.disco_b200_abi_version() == _lib.ABI_VERSION


def test_every_header_symbol_is_exported_and_bound():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 12
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes binding"
    assert set(_lib.SIGNATURES) == set(syms)


def test_every_export_is_declared_in_the_header():
    """export -> header: the library exports no disco_b200_* entry point the header does not declare."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.split() and line.split()[-1].startswith("disco_b200_")}
    assert exported, "no disco_b200_* exports found"
    assert exported == set(declared_symbols()), exported ^ set(declared_symbols())


def test_layout_validation_matches_shard_layout():
    # ShardLayout rules (shard.py:38-49) enforced by the C side too
    with pytest.raises(LayoutError, match="not divisible"):
        _lib.workspace_bytes(8, 4, 3, 0)
    with pytest.raises(LayoutError):
        _lib.workspace_bytes(8, 4, 2, 2)
    with pytest.raises(LayoutError):
        _lib.workspace_bytes(8, 4, 0, 0)
    with pytest.raises(LayoutError):
        _lib.workspace_bytes(0, 4, 1, 0)
    with pytest.raises(ShapeError):
        _lib.workspace_bytes(8, 0, 1, 0)


@pytest.mark.parametrize("B,N,expect", [(32768, 1, (8, 8)), (32768, 2, (8, 4)), (32768, 4, (8, 2)),
                                         (32768, 8, (8, 1)), (1024, 2, (8, 4)), (12, 3, (3, 1)),
                                         (8, 2, (2, 1)), (30000, 2, (2, 1)), (196608, 8, (8, 1))])
def test_canonical_chunking(B, N, expect):
    assert _lib.chunking(B, N) == expect


def test_workspace_regions_are_disjoint_and_aligned():
    B, D, N = 32768, 512, 8
    total = _lib.workspace_bytes(B, D, N, 3)
    spans = []
    for r in range(14):
        off, size = _lib.ws_region(B, D, N, 3, r)
        assert off % 1024 == 0
        assert off + size <= total
        if size:
            spans.append((off, off + size))
    spans.sort()
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 <= b0
    b, Dp = B // N, 512
    assert _lib.ws_region(B, D, N, 3, _lib.R_G)[1] == 2 * b * B * 2          # f16 G, O(B^2/N)
    assert _lib.ws_region(B, D, N, 3, _lib.R_SEND)[1] == N * 2 * b * Dp * 4  # slabs by destination
    assert _lib.ws_region(B, D, N, 3, _lib.R_GATHER)[1] == N * 2 * b * Dp * 2


def test_single_rank_aliases_collective_buffers():
    g = _lib.ws_region(4096, 100, 1, 0, _lib.R_GATHER)
    p = _lib.ws_region(4096, 100, 1, 0, _lib.R_PACK)
    assert g == p
    assert _lib.ws_region(4096, 100, 1, 0, _lib.R_RECV) == _lib.ws_region(4096, 100, 1, 0, _lib.R_SEND)


def test_loss_memory_scales_as_b_squared_over_n():
    # per-GPU loss-scope memory (the f16 G blocks) falls as 1/N at fixed B
    B, D = 65536, 768
    g = [_lib.ws_region(B, D, N, 0, _lib.R_G)[1] for N in (1, 2, 4, 8)]
    assert g[0] == 2 * g[1] == 4 * g[2] == 8 * g[3]


def test_launch_counter_starts_at_zero_without_gpu():
    assert _lib.launch_count() >= 0


@pytest.mark.parametrize("backward", ["dual", "exchange"])
def test_peer_window_geometry(monkeypatch, backward):
    """Peer window = flag block + two parity windows of [2][N*np][b][Dp] f32 (every source's leaves;
    exchange backward only -- the dual backward exchanges no gradients) + two parity areas of this
    rank's published [2][b][Dp] bf16 rows (the peer all-gather) + two of [N][2][b] f32 ce."""
    monkeypatch.setenv("DISCO_BACKWARD", backward)
    out = ctypes.c_int64()
    lib = _lib.load()
    assert lib.disco_b200_peer_handle_bytes() == 64
    # D = 768 (split width: wide + narrow launches) keeps one leaf per canonical chunk like D = 512;
    # B = 3072, N = 3 has no canonical chunks (no stored E, so no dual backward either)
    for B, D, N, leaves in [(32768, 512, 8, 8), (32768, 512, 2, 8), (65536, 768, 4, 8), (3072, 256, 3, 3)]:
        _lib.call("disco_b200_peer_bytes", B, D, N, 0, ctypes.byref(out))
        b, Dp = B // N, (D + 63) // 64 * 64
        dual = backward == "dual" and _lib.path_info(B, D, N, 0) & _lib.PATH_DUAL
        win = 0 if dual else (2 * leaves * b * Dp * 4 + 1023) // 1024 * 1024
        pack = (2 * b * Dp * 2 + 1023) // 1024 * 1024
        ce = (N * 2 * b * 4 + 1023) // 1024 * 1024
        assert out.value == 1024 + 2 * win + 2 * pack + 2 * ce, (B, D, N)
    with pytest.raises(LayoutError):  # nothing to exchange at N = 1
        _lib.call("disco_b200_peer_bytes", 4096, 512, 1, 0, ctypes.byref(out))
    with pytest.raises(LayoutError):  # b % 128 != 0
        _lib.call("disco_b200_peer_bytes", 4096 + 64 * 2, 512, 2, 0, ctypes.byref(out))


def test_wavefront_forward_availability():
    """The H2D-pipelined forward needs a single rank and B % 2048 == 0 (whole 256-row tiles per
    wave); waves follow the stats sub-chunks (16 when B % 4096 == 0)."""
    assert _lib.forward_waves(32768, 512, 1, 0) == 16
    assert _lib.forward_waves(4096, 512, 1, 0) == 16
    assert _lib.forward_waves(2048, 64, 1, 0) == 8
    assert _lib.forward_waves(3072, 512, 1, 0) == 0
    assert _lib.forward_waves(32768, 512, 2, 0) == 0


def test_path_info_reports_the_dual_backward(monkeypatch):
    """Geometry only (no GPU): disco_step's backward is the dual one (rank-local H = G_d + G_d'^T
    GEMMs, no gradient reduce-scatter) wherever the forward stores E (B % 1024 == 0, N | 8), at
    every world size; DISCO_BACKWARD=exchange (read per call) selects the exchange backward."""
    from paper_2304_08480_b200 import _lib
    monkeypatch.delenv("DISCO_BACKWARD", raising=False)
    for B, D, N in [(32768, 512, 1), (32768, 512, 8), (65536, 768, 8), (16384, 1024, 1), (1024, 16, 2),
                    (196608, 512, 8)]:
        bits = _lib.path_info(B, D, N)
        assert bits & _lib.PATH_ESTORE and bits & _lib.PATH_DUAL, (B, D, N)
    assert _lib.path_info(32768, 512, 1) & _lib.PATH_WIDE
    assert not _lib.path_info(65536, 768, 8) & _lib.PATH_WIDE
    for B, D, N in [(1000, 100, 1), (96, 24, 3), (3072, 512, 3)]:  # no stored E: recompute + exchange
        assert not _lib.path_info(B, D, N) & (_lib.PATH_ESTORE | _lib.PATH_DUAL), (B, D, N)
    assert not _lib.path_info(4096, 4096, 1) & _lib.PATH_DUAL  # Dp > 2048: the fixup's row limit
    monkeypatch.setenv("DISCO_BACKWARD", "exchange")
    bits = _lib.path_info(32768, 512, 1)
    assert bits & _lib.PATH_ESTORE and not bits & _lib.PATH_DUAL
