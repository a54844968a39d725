"""ctypes binding of the C ABI declared in include/liger_b200.h.

This is the same binding a maintainer would add on the reference side
(INTEGRATION.md): plain pointers and sizes, a cudaStream_t as void*, int status.
Loading never falls back to anything: if the library is missing the ops raise
ExtensionMissing.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from . import errors

_LOCK = threading.Lock()
_LIB: C.CDLL | None = None

c_i64 = C.c_int64
c_int = C.c_int
c_float = C.c_float
c_size = C.c_size_t
c_void = C.c_void_p
c_i64p = C.POINTER(C.c_int64)
c_fp = C.POINTER(C.c_float)

LK_F32, LK_BF16, LK_F16 = 0, 1, 2
REDUCTIONS = {"none": 0, "mean": 1, "sum": 2}
CASTING = {"llama": 0, "gemma": 1, "none": 2}
LK_ACCUM_AUTO, LK_ACCUM_FP32, LK_ACCUM_WEIGHT_DTYPE = 0, 1, 2


class FlceArgs(C.Structure):
    """Mirror of lk_flce_args (include/liger_b200.h)."""

    _fields_ = [
        ("x", c_void),
        ("weight", c_void),
        ("target", c_void),
        ("bias", c_void),
        ("bt", c_i64),
        ("hidden", c_i64),
        ("vocab", c_i64),
        ("dtype", c_int),
        ("ignore_index", c_i64),
        ("label_smoothing", c_float),
        ("lse_square_scale", c_float),
        ("softcap", c_float),
        ("reduction", c_int),
        ("chunk_rows", c_i64),
        ("loss_rows", c_void),
        ("loss_sum", c_void),
        ("z_loss_rows", c_void),
        ("z_loss_sum", c_void),
        ("grad_x", c_void),
        ("grad_w", c_void),
        ("grad_bias", c_void),
        ("target_stats", c_void),
        ("workspace", c_void),
        ("workspace_bytes", c_size),
        ("stream", c_void),
        ("force_simt", c_int),
        ("mean_count", c_void),
        ("grad_w_accum", c_int),
        ("token_correct_rows", c_void),
        ("predicted_tokens", c_void),
        ("grad_w_slices", c_int),
        ("grad_w_slice_events", c_void),
        ("use_token_scaling", c_int),
        ("ce_weight", c_void),
        ("mean_weight_sum", c_void),
        ("fp32_pieces", c_int),
        ("x_row_index", c_void),
        ("row_limit", c_void),
    ]


# name -> (restype, argtypes); every symbol include/liger_b200.h declares.
SIGNATURES: dict[str, tuple] = {
    "lk_last_error": (C.c_char_p, []),
    "lk_version": (C.c_char_p, []),
    "lk_has_tcgen05": (c_int, []),
    "lk_profile_enable": (None, [c_int]),
    "lk_profile_collect": (c_int, [C.POINTER(C.c_double), c_i64p]),
    "lk_launch_count": (c_i64, []),
    "lk_test_select_path": (c_int, [c_int, c_int]),
    "lk_cross_entropy_workspace_bytes": (c_size, [c_i64]),
    "lk_cross_entropy_fwd_ex": (c_int, [c_void, c_i64, c_void, c_i64, c_i64, c_int, c_i64, c_float, c_float, c_float,
                                        c_int, c_int, c_void, c_void, c_void, c_void, c_void, c_void, c_void, c_void,
                                        c_size, c_void]),
    "lk_flce_workspace_bytes_ex": (c_size, [c_i64, c_i64, c_i64, c_int, c_i64, c_int, c_int]),
    "lk_cross_entropy_fwd": (
        c_int,
        [c_void, c_i64, c_void, c_i64, c_i64, c_int, c_i64, c_float, c_float, c_float, c_int, c_int,
         c_void, c_void, c_void, c_void, c_void, c_size, c_void],
    ),
    "lk_count_targets": (c_int, [c_void, c_i64, c_i64, c_i64, c_void, c_void]),
    "lk_scale_by_device_scalar": (c_int, [c_void, c_i64, c_i64, c_i64, c_int, c_void, c_void]),
    "lk_scale_rows": (c_int, [c_void, c_i64, c_i64, c_i64, c_int, c_void, c_int, c_void]),
    "lk_flce_plan": (c_int, [c_i64, c_i64, c_i64, c_int, c_i64p, c_i64p]),
    "lk_flce_workspace_bytes": (c_size, [c_i64, c_i64, c_i64, c_int, c_i64, c_int]),
    "lk_flce_forward_backward": (c_int, [C.POINTER(FlceArgs)]),
    "lk_flce_workspace_bytes_for": (c_size, [C.POINTER(FlceArgs)]),
    "lk_flce_vp_workspace_bytes": (c_size, [c_i64, c_i64, c_i64, c_int]),
    "lk_flce_vp_logits": (
        c_int,
        [c_void, c_void, c_void, c_i64, c_i64, c_i64, c_i64, c_int, c_i64, c_float, c_void, c_void,
         c_void, c_size, c_void],
    ),
    "lk_flce_vp_backward": (
        c_int,
        [c_void, c_void, c_void, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_i64, c_float, c_float,
         c_float, c_int, c_void, c_void, c_void, c_void, c_void, c_void, c_int, c_void, c_size, c_void],
    ),
    "lk_flce_vp_backward_ex": (
        c_int,
        [c_void, c_void, c_void, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_i64, c_float, c_float,
         c_float, c_int, c_void, c_void, c_void, c_void, c_void, c_void, c_int, c_int, c_void, c_size, c_void],
    ),
    "lk_flce_vp_backward2": (
        c_int,
        [c_void, c_void, c_void, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_i64, c_float, c_float,
         c_float, c_int, c_void, c_void, c_void, c_void, c_void, c_int, c_void, c_int, c_int, c_void, c_size,
         c_void],
    ),
    "lk_flce_vp_combine_stats": (c_int, [c_void, c_i64, c_i64, c_void, c_void]),
    "lk_compact_rows": (c_int, [c_void, c_i64, c_i64, c_void, c_void, c_void, c_void]),
    "lk_gather_rows": (c_int, [c_void, c_i64, c_int, c_void, c_i64, c_void, C.c_uint64, c_void]),
    "lk_peer_alloc": (c_int, [c_int, c_size, C.POINTER(C.c_void_p), c_void]),
    "lk_peer_open": (c_int, [c_int, c_void, C.POINTER(C.c_void_p)]),
    "lk_peer_close": (c_int, [c_int, c_void]),
    "lk_peer_free": (c_int, [c_int, c_void]),
    "lk_peer_allreduce": (c_int, [C.POINTER(C.c_void_p), c_int, c_int, c_i64, c_i64, c_int, C.c_uint64, c_i64,
                                  c_void]),
    "lk_peer_status": (c_int, [c_int, c_void, c_int, C.POINTER(c_int)]),
    "lk_rmsnorm_fwd": (
        c_int, [c_void, c_void, c_void, c_void, c_i64, c_i64, c_float, c_float, c_int, c_int, c_void]
    ),
    "lk_rmsnorm_bwd_workspace_bytes": (c_size, [c_i64, c_i64]),
    "lk_rmsnorm_bwd": (
        c_int,
        [c_void, c_void, c_void, c_void, c_void, c_void, c_i64, c_i64, c_float, c_int, c_int, c_void,
         c_size, c_void],
    ),
    "lk_rope": (
        c_int,
        [c_void, c_void, c_void, c_void, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_int, c_int,
         c_void],
    ),
    "lk_swiglu_fwd": (c_int, [c_void, c_void, c_void, c_i64, c_int, c_void]),
    "lk_swiglu_bwd": (c_int, [c_void, c_void, c_void, c_i64, c_int, c_void]),
    "lk_swiglu_fwd_ex": (c_int, [c_void, c_void, c_void, c_i64, c_float, c_int, c_void]),
    "lk_swiglu_bwd_ex": (c_int, [c_void, c_void, c_void, c_i64, c_float, c_int, c_void]),
    "lk_geglu_fwd": (c_int, [c_void, c_void, c_void, c_i64, c_int, c_void]),
    "lk_geglu_bwd": (c_int, [c_void, c_void, c_void, c_i64, c_int, c_void]),
    "lk_layernorm_fwd": (c_int, [c_void, c_void, c_void, c_void, c_void, c_void, c_i64, c_i64, c_float, c_int,
                                 c_void]),
    "lk_layernorm_bwd_workspace_bytes": (c_size, [c_i64, c_i64]),
    "lk_layernorm_bwd": (c_int, [c_void, c_void, c_void, c_void, c_void, c_void, c_void, c_void, c_i64, c_i64, c_int,
                                 c_void, c_size, c_void]),
    "lk_gemm_test_accum16": (c_int, [c_void, c_void, c_void, c_i64, c_i64, c_i64, c_int, c_int, c_int, c_void, c_size,
                                     c_void]),
    "lk_gemm_test": (
        c_int, [c_void, c_void, c_void, c_i64, c_i64, c_i64, c_int, c_int, c_int, c_void, c_size, c_void]
    ),
}


def lib_path() -> Path:
    from ._build import LIB_PATH

    return LIB_PATH


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building in-tree if needed) the sm_100a library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    with _LOCK:
        if _LIB is not None:
            return _LIB
        from . import _build

        path = _build.LIB_PATH
        if build_if_missing and _build.is_stale():
            try:
                _build.build()
            except Exception as exc:  # pragma: no cover - only without nvcc
                if not path.exists():
                    raise errors.ExtensionMissing(f"cannot build {path}: {exc}") from exc
        if not path.exists():
            raise errors.ExtensionMissing(f"{path} is missing; run __graft_entry__.build()")
        lib = C.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
        return lib


def check(rc: int) -> None:
    """Map an lk_status code to the reference's exception taxonomy."""
    if rc == 0:
        return
    msg = load().lk_last_error().decode(errors="replace")
    raise errors.STATUS.get(rc, RuntimeError)(msg)


# Test-only path knobs (include/liger_b200.h lk_test_select_path): 0 = the product path.
PATH_CTA_GROUP, PATH_FLCE_FINALIZE, PATH_FLCE_SEPARATE_CAST, PATH_CE_IMPL, PATH_NORM_IMPL, PATH_DW_ACCUM16 = range(6)


class select_path:
    """Context manager for the parity tests: run a block on an alternative kernel path."""

    def __init__(self, knob: int, value: int):
        self.knob, self.value = knob, value

    def __enter__(self):
        self.prev = load().lk_test_select_path(self.knob, self.value)
        if self.prev < 0:
            raise ValueError(f"unknown path knob {self.knob} / value {self.value}")
        return self

    def __exit__(self, *exc):
        load().lk_test_select_path(self.knob, self.prev)
