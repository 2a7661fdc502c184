"""ctypes binding of the C ABI in ``include/ukan_b200.h`` (``libukan_b200.so``).

This module is the exact binding a Python caller of the C ABI writes; there is no other
implementation behind it.  If the shared library is missing or no CUDA device is present the
product path raises — it never falls back to a CPU or PyTorch implementation.
"""
from __future__ import annotations

import ctypes
import os

import torch

from .errors import ConfigError, DomainError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UKAN_B200_LIB") or os.path.join(_HERE, "libukan_b200.so")  # override: A/B tooling

UKAN_OK = 0
UKAN_E_ARG = -1
UKAN_E_DEGREE = -2
UKAN_E_GRID = -3
UKAN_E_WORKSPACE = -4
UKAN_E_CAPACITY = -5
UKAN_F32 = 0
UKAN_F64 = 1

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_F64 = ctypes.c_double
_INT = ctypes.c_int
_F32 = ctypes.c_float

# name -> (restype, argtypes); mirrors include/ukan_b200.h one to one
SIGNATURES: dict[str, tuple] = {
    "ukan_version": (_INT, []),
    "ukan_launch_count": (_I64, []),
    "ukan_basis_matrix": (_INT, [_INT, _P]),
    "ukan_kan_forward": (_INT, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT, _F64, _F64, _P, _P]),
    "ukan_kan_forward_workspace_size": (_I64, [_I64, _I64, _I64, _I64, _INT]),
    "ukan_kan_forward_ws": (_INT, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT, _F64, _F64, _P, _P, _I64, _P]),
    "ukan_kan_backward": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT,
                                 _F64, _F64, _P]),
    "ukan_kan_backward_workspace_size": (_I64, [_I64, _I64, _I64, _I64, _INT]),
    "ukan_kan_backward_ws": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT,
                                    _F64, _F64, _P, _I64, _P]),
    "ukan_kan_backward_ws2": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT, _F64, _F64,
                                     _P, _I64, _INT, _P]),
    "ukan_kan_backward_prep": (_INT, [_P, _P, _I64, _I64, _I64, _I64, _INT, _F64, _F64, _P, _I64, _P, _P]),
    "ukan_kan_backward_part_supported": (_INT, [_I64, _I64, _I64, _I64, _INT]),
    "ukan_kan_backward_part": (_INT, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT, _F64, _F64, _P, _I64,
                                      _I64, _I64, _INT, _P]),
    "ukan_kan_naive_forward": (_INT, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT, _F64, _F64, _P]),
    "ukan_kan_naive_backward": (_INT, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT, _F64, _F64, _P]),
    "ukan_kan_jvp_forward": (_INT, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT, _F64, _F64, _P]),
    "ukan_kan_jvp_backward": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT,
                                     _F64, _F64, _P]),
    "ukan_ukan_jvp_forward": (_INT, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _INT, _F64, _P]),
    "ukan_ukan_jvp_backward": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT,
                                      _F64, _P]),
    "ukan_adam_step_dev": (_INT, [_P, _P, _P, _P, _I64, _P, _F64, _F64, _F64, _F64, _P, _P, _P, _P]),
    "ukan_kan_locate": (_INT, [_P, _P, _P, _I64, _I64, _I64, _F64, _F64, _P]),
    "ukan_ukan_keys_workspace_size": (_I64, [_I64, _I64, _I64]),
    "ukan_ukan_build_keys": (_INT, [_P, _I64, _I64, _INT, _F64, _P, _P, _P, _P, _I64, _P, _I64, _P, _P,
                                    _P, _P]),
    "ukan_ukan_cg_input": (_INT, [_P, _P, _P, _P, _I64, _I64, _I64, _P]),
    "ukan_gemm_bias_act": (_INT, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _INT, _P]),
    "ukan_gemm_nt": (_INT, [_P, _P, _P, _I64, _I64, _I64, _P]),
    "ukan_gemm_tn": (_INT, [_P, _P, _P, _P, _I64, _I64, _I64, _P]),
    "ukan_gemm_tn_tf32x3_probe": (_INT, [_P, _P, _P, _I64, _I64, _I64, _P]),
    "ukan_silu_backward": (_INT, [_P, _P, _P, _I64, _P]),
    "ukan_gemm_f64": (_INT, [_INT, _P, _INT, _P, _INT, _P, _INT, _P, _P, _P, _P, _I64, _I64, _I64, _P]),
    "ukan_ukan_emb_backward": (_INT, [_P, _P, _P, _I64, _I64, _I64, _P]),
    "ukan_ukan_forward": (_INT, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _INT, _F64, _P]),
    "ukan_ukan_backward_workspace_size": (_I64, [_I64, _I64, _I64, _I64, _INT]),
    "ukan_ukan_forward_dense_workspace_size": (_I64, [_I64, _I64, _I64, _I64, _INT]),
    "ukan_ukan_forward_dense": (_INT, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT, _F64, _P, _I64, _P]),
    "ukan_ukan_backward2_workspace_size": (_I64, [_I64, _I64, _I64, _I64, _I64, _INT]),
    "ukan_ukan_backward2": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _INT, _F64, _P,
                                   _I64, _P]),
    "ukan_ukan_backward_dense_workspace_size": (_I64, [_I64, _I64, _I64, _I64, _I64, _INT]),
    "ukan_ukan_backward_dense": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _INT, _F64,
                                        _P, _I64, _P]),
    "ukan_ukan_backward": (_INT, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _INT, _F64,
                                  _P, _I64, _P]),
    "ukan_softmax_xent": (_INT, [_P, _P, _P, _P, _I64, _I64, _I64, _F64, _P, _P]),
    "ukan_mse": (_INT, [_P, _P, _P, _P, _I64, _I64, _P]),
    "ukan_adam_step": (_INT, [_P, _P, _P, _P, _I64, _F64, _F64, _F64, _F64, _F64, _I64, _P, _P]),
    "ukan_sgd_step": (_INT, [_P, _P, _I64, _F64, _P, _P]),
    "ukan_fill_f32": (_INT, [_P, _I64, _F32, _P]),
}

_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libukan_b200.so and declare every exported symbol's signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2408_11200_b200.csrc.build` "
            "(the CUDA extension is required; there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    older_build = bool(os.environ.get("UKAN_B200_LIB"))  # A/B tooling may load an older build
    for name, (res, args) in SIGNATURES.items():
        if older_build and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def require_cuda(*tensors: torch.Tensor) -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2408_11200_b200 kernels need a CUDA (sm_100a) device; "
                           "there is no CPU fallback")
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise RuntimeError("all tensors must live on the CUDA device")


def require_params(device, *params: torch.Tensor | None) -> None:
    """Layer parameters go to the kernels as raw pointers: they must be fp32, contiguous and on
    the input's device (a float64 or strided tensor would be read as garbage)."""
    for t in params:
        if t is None:
            continue
        if t.dtype != torch.float32 or not t.is_contiguous() or t.device != device:
            raise ConfigError(f"layer parameters must be contiguous float32 tensors on {device}; got "
                              f"{t.dtype}, contiguous={t.is_contiguous()}, device={t.device}")


def ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_ptr(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def check(rc: int, what: str) -> None:
    if rc == UKAN_OK:
        return
    if rc == UKAN_E_DEGREE:
        raise DomainError(f"{what}: spline degree must be in [0, 10]")
    if rc == UKAN_E_GRID:
        raise ConfigError(f"{what}: invalid grid (need g_min < g_max, G >= 1, delta_g > 0)")
    if rc < 0:
        raise ValueError(f"{what}: argument error (code {rc})")
    raise RuntimeError(f"{what}: CUDA error {rc}")
