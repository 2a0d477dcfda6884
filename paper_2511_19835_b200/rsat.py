"""RSAT tensor files (reference rsat.py:1-62) and their ingest onto the GPU.

Format: magic ``RSAT``, version u8 = 1, dtype u8 (0 = f32, 1 = f64), rank u8,
``rank`` little-endian u64 dims, then row-major little-endian data.
``read_rsat`` / ``write_rsat`` mirror the reference (same bytes, same
``IoError`` cases).  ``read_rsat_to_device`` reads the payload straight into
page-locked memory and copies it to the GPU (optionally casting to bf16 there),
and ``load_problem`` builds an ``AttentionProblem`` from the harness's
problem-path manifest (harness.py:151-170) on the device, ready for the
pipeline -- the ingest half of running real model Q/K/V dumps.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import IoError

MAGIC = b"RSAT"
VERSION = 1
_DTYPE_CODES = {0: np.dtype("<f4"), 1: np.dtype("<f8")}
_CODE_FOR = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}


def write_rsat(path, array: np.ndarray) -> None:
    """Write a float32/float64 array of any rank to an RSAT file (atomically). rsat.py:17-35."""
    arr = np.asarray(array)
    if arr.dtype not in _CODE_FOR:
        raise IoError(f"RSAT stores float32/float64 only, got {arr.dtype}")
    path = Path(path)
    payload = bytearray()
    payload += MAGIC
    payload += struct.pack("<BBB", VERSION, _CODE_FOR[arr.dtype], arr.ndim)
    payload += struct.pack(f"<{arr.ndim}Q", *arr.shape)
    payload += np.ascontiguousarray(arr).astype(arr.dtype.newbyteorder("<")).tobytes()
    tmp = path.with_name(path.name + ".tmp")
    try:
        tmp.write_bytes(payload)
        tmp.replace(path)
    except OSError as exc:
        raise IoError(f"cannot write {path}: {exc}") from exc


def _header(path: Path, raw: bytes, size: int):
    if size < 7 or raw[:4] != MAGIC:
        raise IoError(f"{path} is not an RSAT file")
    version, dtype_code, rank = struct.unpack_from("<BBB", raw, 4)
    if version != VERSION:
        raise IoError(f"{path}: unsupported RSAT version {version}")
    if dtype_code not in _DTYPE_CODES:
        raise IoError(f"{path}: unknown dtype code {dtype_code}")
    header_end = 7 + 8 * rank
    if len(raw) < header_end:
        raise IoError(f"{path}: truncated RSAT header")
    dims = struct.unpack_from(f"<{rank}Q", raw, 7)
    dtype = _DTYPE_CODES[dtype_code]
    count = 1
    for dim in dims:
        count *= dim
    expected = header_end + count * dtype.itemsize
    if size != expected:
        raise IoError(f"{path}: expected {expected} bytes, got {size}")
    return dims, dtype, count, header_end


def read_rsat(path) -> np.ndarray:
    """Read an RSAT file back into a numpy array. rsat.py:38-62."""
    path = Path(path)
    try:
        raw = path.read_bytes()
    except OSError as exc:
        raise IoError(f"cannot read {path}: {exc}") from exc
    dims, dtype, count, header_end = _header(path, raw, len(raw))
    data = np.frombuffer(raw, dtype=dtype, count=count, offset=header_end)
    return data.reshape(dims).astype(dtype.newbyteorder("="))


def read_rsat_to_device(path, device=None, dtype=None):
    """Read an RSAT file into page-locked host memory and copy it to the GPU.
    ``dtype`` (e.g. ``torch.bfloat16``) casts on the device after the copy."""
    import torch

    from .pipeline import _device
    path = Path(path)
    dev = torch.device(device) if device is not None else _device()
    try:
        with open(path, "rb") as f:
            size = path.stat().st_size
            head = f.read(min(size, 7 + 8 * 255))
            dims, np_dtype, count, header_end = _header(path, head, size)
            torch_dtype = torch.float32 if np_dtype.itemsize == 4 else torch.float64
            staging = torch.empty(count, dtype=torch_dtype).pin_memory()
            f.seek(header_end)
            view = staging.numpy().view(np.uint8)
            if f.readinto(memoryview(view)) != count * np_dtype.itemsize:
                raise IoError(f"{path}: short read")
    except OSError as exc:
        raise IoError(f"cannot read {path}: {exc}") from exc
    out = staging.to(dev, non_blocking=True).view(*dims)
    return out.to(dtype) if dtype is not None else out


def load_problem(paths: dict, device=None, dtype=None):
    """``AttentionProblem`` on the GPU from the harness's problem-path manifest
    ({q_video, q_text, k, v, block[, d, grid_dims]}; harness.py:151-170)."""
    from .core import AttentionProblem
    if "block" not in paths:
        raise IoError("problem paths are missing 'block'")
    arrays = {}
    for name in ("q_video", "q_text", "k", "v"):
        if name not in paths:
            raise IoError(f"problem paths are missing {name!r}")
        p = Path(paths[name])
        if not p.exists():
            raise IoError(f"missing input file: {p}")
        arrays[name] = read_rsat_to_device(p, device, dtype)
    grid_dims = tuple(paths["grid_dims"]) if paths.get("grid_dims") else None
    return AttentionProblem(q_video=arrays["q_video"], q_text=arrays["q_text"], k=arrays["k"],
                            v=arrays["v"], d=int(paths.get("d", arrays["q_video"].shape[1])),
                            block=int(paths["block"]), grid_dims=grid_dims)
