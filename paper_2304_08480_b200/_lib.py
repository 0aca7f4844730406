"""ctypes binding of the C ABI in include/disco_b200.h.

The shared library is built in-tree (``python -m paper_2304_08480_b200.build``
or ``__graft_entry__.build()``) as ``paper_2304_08480_b200/_disco_b200.so``.
There is no fallback: if the library is missing every entry point raises.
"""

import ctypes
import os
import threading

from .errors import DomainError, LayoutError, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_disco_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "disco_b200.h")

ABI_VERSION = 3

# status codes (disco_status)
OK, SHAPE, LAYOUT, DOMAIN, NONFINITE, CUDA = 0, 1, 2, 3, 4, 5

# dtype codes (disco_dtype)
F32, BF16, F64, F16 = 0, 1, 2, 3

# workspace regions (disco_region)
R_PACK, R_GATHER, R_FEAT, R_FEAT16, R_STATS, R_ROWS, R_CE, R_CE_ALL, R_G, R_XPART, R_SEND, R_RECV, \
    R_INTRA, R_STATUS, R_SCALE, R_RDOT, R_RDOT_ALL, R_XCHG, R_XALL, R_QCOL, R_FIX = range(21)

_i64 = ctypes.c_int64
_int = ctypes.c_int
_vp = ctypes.c_void_p
_f32 = ctypes.c_float

# name -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES = {
    "disco_b200_abi_version": [],
    "disco_b200_set_experiment_flags": [_int],
    "disco_b200_last_error": [],
    "disco_b200_launch_count": [],
    "disco_b200_workspace_bytes": [_i64, _i64, _int, _int, ctypes.POINTER(_i64)],
    "disco_b200_ws_region": [_i64, _i64, _int, _int, _int, ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
    "disco_b200_chunking": [_i64, _int, ctypes.POINTER(_int), ctypes.POINTER(_int)],
    "disco_b200_pack": [_vp, _i64, _i64, _int, _int, _vp, _vp, _i64, _i64, _int, _int, _vp],
    "disco_b200_pack_rows": [_vp, _i64, _i64, _int, _int, _vp, _vp, _i64, _i64, _int, _int, _i64, _i64, _vp],
    "disco_b200_forward": [_vp, _i64, _i64, _int, _int, _f32, _vp],
    "disco_b200_forward_waves": [_i64, _i64, _int, _int, ctypes.POINTER(_int)],
    "disco_b200_path_info": [_i64, _i64, _int, _int, ctypes.POINTER(_int)],
    "disco_b200_forward_wave": [_vp, _i64, _i64, _int, _int, _f32, _int, _vp],
    "disco_b200_forward_streamed": [_vp, _i64, _i64, _int, _int, _f32, ctypes.c_uint32, ctypes.c_double, _vp],
    "disco_b200_h2d_streamed": [_vp, _i64, _i64, _int, _int, _vp, _vp, ctypes.c_uint32, _vp],
    "disco_b200_signal_wave": [_vp, _i64, _i64, _int, _int, _int, ctypes.c_uint32, _vp],
    "disco_b200_forward_finish": [_vp, _i64, _i64, _int, _int, _vp],
    "disco_b200_backward_grad": [_vp, _i64, _i64, _int, _int, _f32, _vp],
    "disco_b200_backward_cross": [_vp, _i64, _i64, _int, _int, _vp],
    "disco_b200_backward_intra": [_vp, _i64, _i64, _int, _int, _vp],
    "disco_b200_backward_fused": [_vp, _i64, _i64, _int, _int, _vp],
    "disco_b200_combine": [_vp, _i64, _i64, _int, _int, _f32, _int, _vp, _vp, _i64, _vp],
    "disco_b200_backward_rows": [_vp, _i64, _i64, _int, _int, _i64, _i64, _vp],
    "disco_b200_combine_rows": [_vp, _i64, _i64, _int, _int, _f32, _int, _i64, _i64, _vp, _vp, _i64, _vp],
    "disco_b200_peer_bytes": [_i64, _i64, _int, _int, ctypes.POINTER(_i64)],
    "disco_b200_peer_handle_bytes": [],
    "disco_b200_peer_alloc": [_i64, ctypes.POINTER(_vp), _vp],
    "disco_b200_peer_open": [_vp, ctypes.POINTER(_vp)],
    "disco_b200_peer_close": [_vp],
    "disco_b200_peer_free": [_vp],
    "disco_b200_peer_publish": [_vp, _i64, _i64, _int, _int, ctypes.POINTER(ctypes.c_uint64), _int, ctypes.c_uint32,
                                _vp],
    "disco_b200_peer_gather": [_vp, _i64, _i64, _int, _int, ctypes.POINTER(ctypes.c_uint64), _int, ctypes.c_uint32,
                               ctypes.c_double, _vp],
    "disco_b200_forward_gathered": [_vp, _i64, _i64, _int, _int, _f32, _vp],
    "disco_b200_peer_gather_streamed": [_vp, _i64, _i64, _int, _int, ctypes.POINTER(ctypes.c_uint64), _int,
                                        ctypes.c_uint32, _vp],
    "disco_b200_forward_peer_streamed": [_vp, _i64, _i64, _int, _int, _f32, ctypes.c_uint32, ctypes.c_double, _vp],
    "disco_b200_backward_peer": [_vp, _i64, _i64, _int, _int, ctypes.POINTER(ctypes.c_uint64), _int,
                                 ctypes.c_uint32, _vp],
    "disco_b200_loss_peer": [_vp, _i64, _i64, _int, _int, _vp, _int, _vp],
    "disco_b200_combine_peer": [_vp, _i64, _i64, _int, _int, _f32, _int, _vp, _int, ctypes.c_uint32,
                                ctypes.c_double, _vp, _vp, _i64, _vp],
    "disco_b200_clock_probe": [_vp, _i64, _i64, _int, _int, ctypes.POINTER(ctypes.c_double)],
    "disco_b200_contribution": [_vp, _i64, _i64, _int, _int, _f32, _int, _vp, _vp, _i64, _vp],
    "disco_b200_loss": [_vp, _i64, _i64, _int, _int, _int, _vp],
    "disco_b200_logit_scale_rows": [_vp, _i64, _i64, _int, _int, _vp, _vp, _i64, _vp],
    "disco_b200_logit_scale_grad": [_vp, _i64, _i64, _int, _int, _f32, _vp],
    "disco_b200_dual_prep": [_vp, _i64, _i64, _int, _int, _int, _vp],
    "disco_b200_backward_dual": [_vp, _i64, _i64, _int, _int, _i64, _i64, _vp],
    "disco_b200_combine_dual": [_vp, _i64, _i64, _int, _int, _f32, _i64, _i64, _vp, _vp, _i64, _vp],
    "disco_b200_dual_fixup": [_vp, _i64, _i64, _int, _int, _f32, _int, _vp, _vp, _i64, _vp],
    "disco_b200_forward_streamed_split": [_vp, _i64, _i64, _int, _int, _f32, ctypes.c_uint32, ctypes.c_double, _int,
                                          _vp],
    "disco_b200_forward_rect": [_vp, _i64, _i64, _int, _int, _f32, _int, _i64, _i64, _int, _int, _vp],
    "disco_b200_stats_rows": [_vp, _i64, _i64, _int, _int, _int, _i64, _i64, _vp],
    "disco_b200_dual_prep_dir": [_vp, _i64, _i64, _int, _int, _int, _int, _vp],
    "disco_b200_backward_dual_dir": [_vp, _i64, _i64, _int, _int, _int, _i64, _i64, _vp],
    "disco_b200_combine_dual_dir": [_vp, _i64, _i64, _int, _int, _int, _f32, _i64, _i64, _vp, _vp, _i64, _vp],
    "disco_b200_finish_dual_l2norm": [_vp, _i64, _i64, _int, _int, _f32, _int, _vp, _i64, _vp, _i64, _vp, _vp, _i64,
                                      _vp, _vp, _i64, _vp, _vp],
    "disco_b200_l2norm_rows": [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _vp],
    "disco_b200_l2norm_rows_backward": [_vp, _i64, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp],
}
_RESTYPES = {"disco_b200_last_error": ctypes.c_char_p, "disco_b200_launch_count": _i64}

_lock = threading.Lock()
_lib = None


class NativeLibraryMissing(RuntimeError):
    """The CUDA extension is not built; there is deliberately no CPU fallback."""


def load():
    """Load (once) and return the ctypes handle; raises if the .so is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not found: build it with `python -m paper_2304_08480_b200.build` "
                "(no CPU fallback exists for the DisCo loss path)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, _int)
        if lib.disco_b200_abi_version() != ABI_VERSION:
            raise NativeLibraryMissing("ABI version mismatch: rebuild the extension")
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().disco_b200_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Map a disco_status code to the reference exception taxonomy (errors.py)."""
    if rc == OK:
        return
    msg = last_error()
    if rc == SHAPE:
        raise ShapeError(msg)
    if rc == LAYOUT:
        raise LayoutError(msg)
    if rc == DOMAIN:
        raise DomainError(msg)
    if rc == NONFINITE:
        raise ValueError(f"{msg} (contains non-finite entries)")
    raise RuntimeError(f"disco_b200 CUDA error: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def workspace_bytes(B: int, D: int, world: int, rank: int) -> int:
    out = _i64()
    call("disco_b200_workspace_bytes", B, D, world, rank, ctypes.byref(out))
    return out.value


def ws_region(B: int, D: int, world: int, rank: int, region: int):
    off, size = _i64(), _i64()
    call("disco_b200_ws_region", B, D, world, rank, region, ctypes.byref(off), ctypes.byref(size))
    return off.value, size.value


def chunking(B: int, world: int):
    nchunk, cpr = _int(), _int()
    call("disco_b200_chunking", B, world, ctypes.byref(nchunk), ctypes.byref(cpr))
    return nchunk.value, cpr.value


def forward_waves(B: int, D: int, world: int, rank: int) -> int:
    """Waves of the H2D-pipelined forward (0: shape not wavefront-capable)."""
    out = _int()
    call("disco_b200_forward_waves", B, D, world, rank, ctypes.byref(out))
    return out.value


PATH_ESTORE, PATH_WIDE, PATH_DUAL = 1, 2, 4


def path_info(B: int, D: int, world: int, rank: int = 0) -> int:
    """disco_b200_path_info bit mask (PATH_*): which kernels this geometry runs right now."""
    out = _int()
    call("disco_b200_path_info", B, D, world, rank, ctypes.byref(out))
    return out.value


def clock_probe(plan) -> dict:
    """SM clock (MHz) the last logits kernel / backward GEMM ran at (CTA 0 stamps)."""
    out = (ctypes.c_double * 3)()
    call("disco_b200_clock_probe", *plan.args, out)
    return {"logits_fwd": round(out[0], 1), "gemm_backward": round(out[1], 1), "drain_cycles_per_unit": round(out[2])}


def launch_count() -> int:
    """Kernels launched by the library so far in this process."""
    return int(load().disco_b200_launch_count())
