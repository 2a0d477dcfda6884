"""``torch.ops.rsa_b200.*``: the hot path as registered PyTorch operators.

The registration is C++ (``csrc/torch_ops.cpp``, ``TORCH_LIBRARY(rsa_b200)``,
built into ``librsa_b200_torch.so`` over the C ABI of ``librsa_b200.so``),
with CUDA and Meta kernels, so the ops trace under ``torch.compile`` and pass
``torch.library.opcheck``.  Importing this module loads that library; without
it the import raises NativeError (no Python fallback).

    torch.ops.rsa_b200.rectified_sparse_attention(q, k, v, num_text_tokens, block=128,
        top_k_fraction=0.1, weight_threshold=0.0, adjacency_radius=0,
        force_text_blocks=False, variant="sparse-rectified") -> Tensor
    torch.ops.rsa_b200.rectified_sparse_attention_status(...) -> (Tensor, Tensor int32[4])

q/k/v are ``[..., T, d]`` (the last ``num_text_tokens`` rows text; reference
core.py:6-8), config as SparsityConfig (masks.py:30-33), variant as VARIANTS
(rectify.py:23-24).  The first op checks the device flags eagerly (one stream
sync, like the reference's eager checks); the second returns them for
``raise_for_status``.  Operator errors surface as RuntimeError whose message
starts with the reference exception's class name; :func:`rectified_sparse_attention`
here re-raises them as those classes (errors.py:4-45).
"""

from __future__ import annotations

import os
from pathlib import Path

import torch

from . import errors
from ._native import lib as _load_native
from .errors import NativeError

TORCH_LIB_PATH = Path(os.environ.get("RSA_B200_TORCH_LIB",
                                     Path(__file__).resolve().parent / "librsa_b200_torch.so"))


def _load() -> None:
    if hasattr(torch.ops.rsa_b200, "rectified_sparse_attention"):
        return
    _load_native()    # the C ABI library it links against (raises if missing)
    if not TORCH_LIB_PATH.exists():
        raise NativeError(f"{TORCH_LIB_PATH} is missing: run `python -m paper_2511_19835_b200.build`")
    torch.ops.load_library(str(TORCH_LIB_PATH))


_load()


def typed_error(exc: RuntimeError) -> Exception:
    """The reference exception class an operator error names, else the error."""
    msg = str(exc)
    for line in msg.splitlines():
        name, sep, rest = line.partition(": ")
        cls = getattr(errors, name.strip(), None) if sep else None
        if isinstance(cls, type) and issubclass(cls, errors.RectAttnError):
            return cls(rest)
    return exc


def rectified_sparse_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, num_text_tokens: int,
                               block: int = 128, top_k_fraction: float = 0.1, weight_threshold: float = 0.0,
                               adjacency_radius: int = 0, force_text_blocks: bool = False,
                               variant: str = "sparse-rectified") -> torch.Tensor:
    """``torch.ops.rsa_b200.rectified_sparse_attention`` with the reference's
    exception classes."""
    try:
        return torch.ops.rsa_b200.rectified_sparse_attention(q, k, v, num_text_tokens, block, top_k_fraction,
                                                             weight_threshold, adjacency_radius,
                                                             force_text_blocks, variant)
    except RuntimeError as exc:
        raise typed_error(exc) from exc
