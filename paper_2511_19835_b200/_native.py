"""ctypes binding of librsa_b200.so (include/rsa_b200.h).

The library is the product: there is no Python or CPU fallback.  ``lib()``
raises NativeError when the shared object is missing or fails to load, and
every call converts an rsa_status into the reference's exception classes.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import STATUS_TO_ERROR, NativeError

LIB_PATH = Path(os.environ.get("RSA_B200_LIB", Path(__file__).resolve().parent / "librsa_b200.so"))

DTYPE_CODES = {"bfloat16": 0, "float32": 1, "float64": 2}
VARIANT_CODES = {"full": 0, "sparse-unrectified": 1, "sparse-rectified": 2,
                 "sparse-rectified-no-gapr": 3, "compensate-all": 4}
KERNEL_CODES = {"auto": 0, "tcgen05": 1, "simt": 2, "tcgen05-persistent": 3, "tcgen05-pingpong": 4}

EXPORTS = ("rsa_plan", "rsa_workspace_layout_query", "rsa_workspace_size", "rsa_pool",
           "rsa_select", "rsa_attention", "rsa_forward", "rsa_forward_strided", "rsa_forward_host",
           "rsa_block_sparse_attention",
           "rsa_text_full_attention", "rsa_morton_permutation", "rsa_permute_rows",
           "rsa_permuted_buffer_size", "rsa_forward_permuted", "rsa_diagnostics_scratch_size", "rsa_diagnostics",
           "rsa_dense_reference_scratch_size", "rsa_dense_reference",
           "rsa_check_device_status", "rsa_accumulate_status", "rsa_status_from_flags",
           "rsa_last_launch_count",
           "rsa_last_error", "rsa_version")


class Shape(C.Structure):
    _fields_ = [("heads", C.c_int64), ("t_video", C.c_int64), ("t_text", C.c_int64),
                ("head_dim", C.c_int64), ("block", C.c_int64), ("dtype", C.c_int32),
                ("kernel", C.c_int32), ("flags", C.c_int32), ("reserved", C.c_int32)]


SHAPE_RAGGED_VIDEO = 1   # rsa_shape.flags: final video block may hold < block tokens


class Config(C.Structure):
    _fields_ = [("top_k_fraction", C.c_double), ("weight_threshold", C.c_double),
                ("adjacency_radius", C.c_int32), ("force_text_blocks", C.c_int32),
                ("variant", C.c_int32), ("reserved", C.c_int32)]


class Grid(C.Structure):
    _fields_ = [("n_q", C.c_int64), ("n_kv", C.c_int64), ("n_text_blocks", C.c_int64),
                ("last_text_block_len", C.c_int64), ("n_cols", C.c_int64),
                ("last_video_block_len", C.c_int64)]


LAYOUT_FIELDS = ("q_pool", "q_def", "k_cat", "k_def", "v_pool", "scores", "a_pool", "mask_bits",
                 "r", "r_eff", "comp", "kv_count", "kv_list", "tile_count", "tile_list", "v_t", "text_part", "text_ml", "a_applied",
                 "status", "total")


class Layout(C.Structure):
    _fields_ = [(n, C.c_size_t) for n in LAYOUT_FIELDS]


class TensorLayout(C.Structure):
    """rsa_layout: element strides of strided Q/K/V/O (head_dim contiguous)."""
    _fields_ = [("heads_per_batch", C.c_int64), ("token_stride", C.c_int64), ("head_stride", C.c_int64),
                ("batch_stride", C.c_int64)]


_LIB = None


def lib() -> C.CDLL:
    """Load the CUDA library once; fail loudly if it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        raise NativeError(f"{LIB_PATH} is missing: run `python -m paper_2511_19835_b200.build` "
                          f"(there is no CPU fallback)")
    try:
        handle = C.CDLL(str(LIB_PATH))
    except OSError as exc:
        raise NativeError(f"cannot load {LIB_PATH}: {exc}") from exc
    P = C.c_void_p
    sigs = {
        "rsa_plan": ([C.POINTER(Shape), C.POINTER(Config), C.POINTER(Grid)], C.c_int),
        "rsa_workspace_layout_query": ([C.POINTER(Shape), C.POINTER(Layout)], C.c_int),
        "rsa_workspace_size": ([C.POINTER(Shape)], C.c_size_t),
        "rsa_pool": ([C.POINTER(Shape), P, P, P, P, P], C.c_int),
        "rsa_select": ([C.POINTER(Shape), C.POINTER(Config), P, P], C.c_int),
        "rsa_attention": ([C.POINTER(Shape), C.POINTER(Config), P, P, P, P, P, P, P], C.c_int),
        "rsa_forward": ([C.POINTER(Shape), C.POINTER(Config), P, P, P, P, P, P, P], C.c_int),
        "rsa_forward_strided": ([C.POINTER(Shape), C.POINTER(Config), C.POINTER(TensorLayout),
                                 C.POINTER(TensorLayout), P, P, P, P, P, P, P], C.c_int),
        "rsa_forward_host": ([C.POINTER(Shape), C.POINTER(Config), P, P, P, P, P, P, P, P, P, P,
                              C.c_int64, P], C.c_int),
        "rsa_block_sparse_attention": ([C.POINTER(Shape), P, P, P, P, P, P, P, P], C.c_int),
        "rsa_text_full_attention": ([C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int32, P, P, P, P, P, P, P], C.c_int),
        "rsa_morton_permutation": ([C.c_int64, C.c_int64, C.c_int64, P], C.c_int),
        "rsa_permute_rows": ([C.POINTER(Shape), P, P, P, C.c_int32, P], C.c_int),
        "rsa_permuted_buffer_size": ([C.POINTER(Shape)], C.c_size_t),
        "rsa_forward_permuted": ([C.POINTER(Shape), C.POINTER(Config), P, P, P, P, P, P, P, P, P], C.c_int),
        "rsa_diagnostics_scratch_size": ([C.POINTER(Shape)], C.c_size_t),
        "rsa_diagnostics": ([C.POINTER(Shape), P, P, P, P, P, P, P, P, P, P, P], C.c_int),
        "rsa_dense_reference_scratch_size": ([C.POINTER(Shape)], C.c_size_t),
        "rsa_dense_reference": ([C.POINTER(Shape), P, P, P, P, P, P], C.c_int),
        "rsa_check_device_status": ([P, P], C.c_int),
        "rsa_accumulate_status": ([P, P, P], C.c_int),
        "rsa_status_from_flags": ([P], C.c_int),
        "rsa_last_launch_count": ([], C.c_int32),
        "rsa_last_error": ([], C.c_char_p),
        "rsa_version": ([], C.c_char_p),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(handle, name)
        fn.argtypes = args
        fn.restype = res
    _LIB = handle
    return handle


def check(status: int) -> None:
    if status != 0:
        msg = lib().rsa_last_error().decode()
        raise STATUS_TO_ERROR.get(status, NativeError)(msg)


def make_shape(heads, t_video, t_text, head_dim, block, dtype: str, kernel: str = "auto",
               ragged_video: bool = False) -> Shape:
    if dtype not in DTYPE_CODES:
        from .errors import ShapeError
        raise ShapeError(f"q/k/v must be bfloat16, float32 or float64, got {dtype}")
    return Shape(int(heads), int(t_video), int(t_text), int(head_dim), int(block),
                 DTYPE_CODES[dtype], KERNEL_CODES[kernel], SHAPE_RAGGED_VIDEO if ragged_video else 0, 0)


def make_config(top_k_fraction, weight_threshold, adjacency_radius, force_text_blocks,
                variant: str) -> Config:
    from .errors import ConfigError
    if variant not in VARIANT_CODES:
        raise ConfigError(f"unknown variant {variant!r}, expected one of {tuple(VARIANT_CODES)}")
    return Config(float(top_k_fraction), float(weight_threshold), int(adjacency_radius),
                  int(bool(force_text_blocks)), VARIANT_CODES[variant], 0)


def plan(shape: Shape, config: Config | None = None) -> Grid:
    g = Grid()
    check(lib().rsa_plan(C.byref(shape), C.byref(config) if config is not None else None, C.byref(g)))
    return g


def layout(shape: Shape) -> dict:
    L = Layout()
    check(lib().rsa_workspace_layout_query(C.byref(shape), C.byref(L)))
    return {n: getattr(L, n) for n in LAYOUT_FIELDS}


def last_launch_count() -> int:
    return int(lib().rsa_last_launch_count())


def version() -> str:
    return lib().rsa_version().decode()
