"""ctypes binding of libjz (include/jz.h).

This is the only place the Python mirror touches native code.  There is no CPU
fallback: if libjz.so is missing, or the current device is not an sm_100 GPU,
every device entry point raises.  Status codes map back to the reference's
exception types (ValueError / IndexError / NonFiniteGradient).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import torch

# JZ_LIB_PATH: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = Path(os.environ.get("JZ_LIB_PATH") or Path(__file__).resolve().parent / "lib" / "libjz.so")

JZ_OK, JZ_EINVAL, JZ_EINDEX, JZ_ECUDA, JZ_EUNSUPPORTED, JZ_ENONFINITE = 0, -1, -2, -3, -4, -5

EPI_F32, EPI_BF16, EPI_RESID, EPI_GELU, EPI_GELU_BWD, EPI_F32_ACC, EPI_BF16_F32 = range(7)
EPI_GELU_DG, EPI_MUL_F16 = 8, 9

_P, _I64, _I32, _F32, _F64, _U64 = C.c_void_p, C.c_int64, C.c_int, C.c_float, C.c_double, C.c_uint64

# name -> argtypes (restype is int status unless listed in _RESTYPE)
PROTOTYPES: dict[str, list] = {
    "jz_device_check": [_I32],
    "jz_gemm_workspace_bytes": [_I64, _I64, _I32],
    "jz_gemm_bf16": [_P, _I64, _I32, _P, _I64, _I32, _P, _I64, _I64, _I64, _I64,
                     _I32, _P, _P, _I64, _P, _I64, _I32, _P, _P],
    "jz_gemm_bf16_colsum": [_P, _I64, _I32, _P, _I64, _I32, _P, _I64, _I64, _I64, _I64,
                            _I32, _P, _P, _I64, _P, _I64, _P, _P],
    "jz_gemm_colsum_parts": [_I64],
    "jz_gemm_bf16_ln_fwd": [_P, _I64, _I32, _P, _I64, _I32, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _F32,
                            _P, _P, _P, _I64, _P],
    "jz_gemm_ln_bwd_parts": [_I64],
    "jz_gemm_bf16_ln_bwd": [_P, _I64, _I32, _P, _I64, _I32, _I64, _I64, _I64, _P, _P, _P, _P, _P, _I32, _P, _P, _I64,
                            _P, _P, _P, _P],
    "jz_row_partials": [_I64],
    "jz_colsum_bf16": [_P, _I64, _I32, _I64, _P, _I32, _P],
    "jz_reduce_partials": [_P, _I32, _I64, _P, _I32, _P],
    "jz_reduce_partials3": [_P, _P, _P, _I32, _I64, _P, _P, _P, _I32, _P],
    "jz_cast_f32_bf16_2d": [_P, _I64, _P, _I64, _I64, _I64, _P],
    "jz_layernorm_fwd": [_P, _I64, _I32, _P, _P, _F32, _P, _P, _P, _P, _I64, _P],
    "jz_layernorm_bwd": [_P, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _I32, _I64, _I32, _I64, _P],
    "jz_layernorm_bwd_bf16dy": [_P, _P, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _I32, _I64, _I32, _I64, _P],
    "jz_ce_fwd_bwd": [_P, _I64, _I32, _P, _P, _P, _F32, _P, _P, _P, _P],
    "jz_finite_check": [_P, _I64, _P, _P],
    "jz_adamw_step": [_P, _P, _P, _P, _I64, _F32, _F32, _F32, _F32, _F32, _F32, _F32, _F32, _F32, _P, _P],
    "jz_philox_mask": [_P, _P, _P, _I32, _I64, _I64, _I64, _I32, _I32, _F64, _P, _P, _P],
    "jz_philox_mask_dev": [_P, _I64, _I64, _I64, _I32, _I32, _F64, _P, _P, _P],
    "jz_adamw_step_dev": [_P, _P, _P, _P, _I64, _P, _P, _P],
    "jz_dyn_embed_fwd": [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32,
                         _I32, _P, _P, _P],
    "jz_embedding_table_bwd": [_P, _P, _I64, _I32, _I32, _P, _I32, _P, _P],
    "jz_dyn_embed_bwd_workspace": [_I64, _I32, _I32, _I32, _I32, _I32, _I32],
    "jz_dyn_embed_bwd": [_P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _I32,
                         _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "jz_attn_spatial_fwd": [_P, _I64, _I32, _I32, _I32, _P, _P, _P, _P],
    "jz_attn_spatial_bwd": [_P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _P, _P, _P, _P],
    "jz_attn_spatial_colsum_parts": [_I64],
    "jz_attn_temporal_colsum_parts": [_I64, _I32],
    "jz_attn_temporal_colsum_parts_t": [_I64, _I32, _I32, _I32],
    "jz_attn_spatial_bwd_workspace_bytes": [_I64, _I32, _I32],
    "jz_attn_temporal_fwd": [_P, _I64, _I32, _I32, _I32, _I32, _P, _P, _P],
    "jz_attn_temporal_bwd": [_P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _P, _P, _P],
    "jz_attn_spatial_small_fwd": [_P, _I64, _I32, _I32, _I32, _P, _P, _P],
    "jz_attn_spatial_small_bwd": [_P, _P, _P, _P, _I64, _I32, _I32, _I32, _P, _P, _P],
    "jz_patchify": [_P, _I32, _I64, _I32, _I32, _I32, _I32, _P, _P, _P],
    "jz_unpatchify": [_P, _I64, _I32, _I32, _I32, _I32, _P, _P, _P],
    "jz_assemble_fwd": [_P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _P, _P],
    "jz_assemble_bwd_workspace": [_I64, _I32, _I32, _I32, _I32],
    "jz_assemble_bwd": [_P, _I64, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P],
    "jz_mean_pool": [_P, _I64, _I32, _I32, _P, _P],
    "jz_mean_pool_bwd": [_P, _I64, _I32, _I32, _P, _P],
    "jz_mse": [_P, _P, _I64, _F32, _P, _P, _P, _P, _P],
    "jz_sum": [_P, _I64, _F64, _P, _P, _P],
    "jz_linear_f32": [_P, _I64, _I32, _P, _I32, _P, _P, _I32, _P],
    "jz_linear_f32_bwd": [_P, _P, _I64, _I32, _I32, _P, _P, _P, _P, _I32, _P],
    "jz_linear_f32_bwd_workspace": [_I64, _I32, _I32],
    "jz_linear_f32_bwd_ws": [_P, _P, _I64, _I32, _I32, _P, _P, _P, _P, _I32, _P, _I64, _P],
    "jz_vq_fwd": [_P, _I64, _I32, _P, _I32, _P, _P, _P, _P],
    "jz_vq_bwd": [_P, _P, _P, _P, _I64, _I32, _I32, _F32, _F32, _P, _P, _P],
    "jz_dyn_embed_frame": [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _P, _P],
    "jz_attn_temporal_decode": [_P, _P, _I64, _I32, _P, _I32, _I32, _I32, _I32, _P, _P],
    "jz_kv_fill": [_P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _P],
    "jz_maskgit_step": [_P, _I64, _I32, _I32, _F32, _P, _P, _P, _I32, _U64, _I32, _P, _P, _P, _P, _P],
}
_RESTYPE = {"jz_gemm_workspace_bytes": _I64, "jz_gemm_ln_bwd_parts": _I64, "jz_linear_f32_bwd_workspace": _I64, "jz_gemm_colsum_parts": _I64, "jz_attn_spatial_colsum_parts": _I64,
            "jz_attn_temporal_colsum_parts": _I64, "jz_attn_temporal_colsum_parts_t": _I64, "jz_attn_spatial_bwd_workspace_bytes": _I64, "jz_dyn_embed_bwd_workspace": _I64, "jz_assemble_bwd_workspace": _I64, "jz_last_error": C.c_char_p,
            "jz_build_info": C.c_char_p}


class NonFiniteGradient(Exception):
    """Raised when a gradient contains NaN/Inf (mirrors deskworld.optim.NonFiniteGradient)."""


_lib = None
_lock = threading.Lock()
_checked_devices: set[int] = set()


def load() -> C.CDLL:
    """Load libjz.so (building it first when sources are present and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists() and os.environ.get("JZ_NO_AUTOBUILD") != "1":
            from . import build as _build
            _build.build()
        if not LIB_PATH.exists():
            raise RuntimeError(f"libjz.so not found at {LIB_PATH}; run `python -m paper_2510_27002_b200.build`")
        lib = C.CDLL(str(LIB_PATH))
        for name, argtypes in PROTOTYPES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPE.get(name, _I32)
        for name in ("jz_last_error", "jz_build_info"):
            fn = getattr(lib, name)
            fn.argtypes = []
            fn.restype = C.c_char_p
        lib.jz_launch_count.argtypes = []
        lib.jz_launch_count.restype = C.c_ulonglong
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    return sorted(PROTOTYPES) + ["jz_last_error", "jz_build_info", "jz_launch_count"]


def launch_count() -> int:
    return int(load().jz_launch_count())


def last_error() -> str:
    return load().jz_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status == JZ_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == JZ_EINVAL:
        raise ValueError(msg)
    if status == JZ_EINDEX:
        raise IndexError(msg)
    if status == JZ_ENONFINITE:
        raise NonFiniteGradient(msg)
    raise RuntimeError(f"libjz status {status}: {msg}")


def ensure_device(device: torch.device | int | None = None) -> int:
    """Fail loudly unless a CUDA sm_100 device is present (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2510_27002_b200 needs a CUDA B200 (sm_100) GPU; none is visible")
    if device is None:
        idx = torch.cuda.current_device()
    elif isinstance(device, int):
        idx = device
    else:
        idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx not in _checked_devices:
        check(load().jz_device_check(idx), "device check")
        _checked_devices.add(idx)
    return idx


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)
