"""torch.library registration of the hot path as ``torch.ops.rsa_b200.*``.

The ops call straight into the C ABI (include/rsa_b200.h) on the current
stream; fake (meta) kernels describe output shapes so the op composes with
tracing.  A model integration replaces its attention call with
``torch.ops.rsa_b200.rectified_sparse_attention(q, k, v, num_text, block, ...)``.
"""

from __future__ import annotations

import torch

from .pipeline import rectified_sparse_attention as _impl

_LIB_NS = "rsa_b200"


@torch.library.custom_op(f"{_LIB_NS}::rectified_sparse_attention", mutates_args=())
def rectified_sparse_attention_op(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                                  num_text_tokens: int, block: int, top_k_fraction: float,
                                  weight_threshold: float, adjacency_radius: int,
                                  force_text_blocks: bool, variant: str) -> torch.Tensor:
    return _impl(q, k, v, num_text_tokens=num_text_tokens, block=block,
                 top_k_fraction=top_k_fraction, weight_threshold=weight_threshold,
                 adjacency_radius=adjacency_radius, force_text_blocks=force_text_blocks,
                 variant=variant)


def _out_like(q, k, v):
    """The real op's output layout: dense in q's dimension order when q/k/v go
    down the strided (no-copy) path, else contiguous."""
    from .pipeline import _dense_like
    strided = (not (q.is_contiguous() and k.is_contiguous() and v.is_contiguous()) and q.dtype == torch.bfloat16
               and q.dim() <= 4 and q.stride() == k.stride() == v.stride() and q.stride(-1) == 1)
    return _dense_like(q) if strided else q.new_empty(q.shape)


@rectified_sparse_attention_op.register_fake
def _(q, k, v, num_text_tokens, block, top_k_fraction, weight_threshold, adjacency_radius,
      force_text_blocks, variant):
    return _out_like(q, k, v)


@torch.library.custom_op(f"{_LIB_NS}::rectified_sparse_attention_status", mutates_args=())
def rectified_sparse_attention_status_op(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                                         num_text_tokens: int, block: int, top_k_fraction: float,
                                         weight_threshold: float, adjacency_radius: int,
                                         force_text_blocks: bool, variant: str
                                         ) -> tuple[torch.Tensor, torch.Tensor]:
    """Non-synchronising form: returns (out, status int32[4]) with the device
    flags of this call; ``raise_for_status(status)`` raises the reference
    exception when the caller next synchronises."""
    from .pipeline import new_status
    status = new_status(q.device)
    out = _impl(q, k, v, num_text_tokens=num_text_tokens, block=block, top_k_fraction=top_k_fraction,
                weight_threshold=weight_threshold, adjacency_radius=adjacency_radius,
                force_text_blocks=force_text_blocks, variant=variant, check_status=False, status=status)
    return out, status


@rectified_sparse_attention_status_op.register_fake
def _(q, k, v, num_text_tokens, block, top_k_fraction, weight_threshold, adjacency_radius,
      force_text_blocks, variant):
    return _out_like(q, k, v), q.new_empty(4, dtype=torch.int32)
