"""Multi-GPU execution of the hot path: one process per GPU.

The reference computes one (batch, head) problem per call (no
cross-head state), so heads are the natural shard: every rank runs the
K1 -> K2 -> K3 pipeline on its own heads with no collective on the data path.

When activations arrive SEQUENCE-sharded (Ulysses / USP style: each rank owns
a contiguous slice of the video tokens of every head, text tokens replicated),
an all-to-all reshuffles sequence shards into head shards before the pipeline
and back after it:

    [B, H, T_v/P, d] per rank --all_to_all--> [B, H/P, T_v, d] per rank
    attention on [B, H/P, T_v + T_t, d] (text rows appended, replicated input)
    [B, H/P, T_v, d] per rank --all_to_all--> [B, H, T_v/P, d] per rank
    text outputs: all_gather over heads (replicated, like the text input)

Collectives go through torch.distributed (NCCL over NVLink on the GPU box,
gloo in the CPU tests).
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def head_range(n_heads: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced head shard [lo, hi) of `rank`."""
    base, extra = divmod(n_heads, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _attention(q, k, v, num_text_tokens: int, **kw):
    from .pipeline import rectified_sparse_attention
    return rectified_sparse_attention(q, k, v, num_text_tokens=num_text_tokens, **kw)


def head_parallel_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, num_text_tokens: int,
                            group=None, gather: bool = False,
                            attn_fn: Callable | None = None, **kw) -> torch.Tensor:
    """q/k/v [B, H, T, d] replicated on every rank (or already this rank's
    head shard when H equals the shard size): each rank runs its heads.
    Returns this rank's [B, H_r, T, d] output, or the full [B, H, T, d] when
    `gather` (all_gather over heads)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    fn = attn_fn or _attention
    lo, hi = head_range(q.shape[1], world, rank)
    out = fn(q[:, lo:hi].contiguous(), k[:, lo:hi].contiguous(), v[:, lo:hi].contiguous(),
             num_text_tokens, **kw)
    if not gather or world == 1:
        return out
    sizes = [head_range(q.shape[1], world, r) for r in range(world)]
    if len({h - l for l, h in sizes}) != 1:
        raise ValueError("gather needs equal head shards (H divisible by the world size)")
    parts = [torch.empty_like(out) for _ in range(world)]
    dist.all_gather(parts, out.contiguous(), group=group)
    return torch.cat(parts, dim=1)


def seq_to_head(x: torch.Tensor, group=None) -> torch.Tensor:
    """Ulysses forward shuffle: [B, H, S/P, d] (this rank's sequence slice of
    every head) -> [B, H/P, S, d] (every token of this rank's heads)."""
    world = dist.get_world_size(group)
    b, h, s_loc, d = x.shape
    if h % world:
        raise ValueError(f"heads ({h}) must be divisible by the world size ({world})")
    hp = h // world
    send = x.reshape(b, world, hp, s_loc, d).permute(1, 0, 2, 3, 4).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    # recv[p] = rank p's sequence slice of my heads
    return recv.permute(1, 2, 0, 3, 4).reshape(b, hp, world * s_loc, d)


def head_to_seq(x: torch.Tensor, group=None) -> torch.Tensor:
    """Inverse shuffle: [B, H/P, S, d] -> [B, H, S/P, d]."""
    world = dist.get_world_size(group)
    b, hp, s, d = x.shape
    if s % world:
        raise ValueError(f"sequence ({s}) must be divisible by the world size ({world})")
    s_loc = s // world
    send = x.reshape(b, hp, world, s_loc, d).permute(2, 0, 1, 3, 4).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    # recv[p] = my sequence slice of rank p's heads
    return recv.permute(1, 0, 2, 3, 4).reshape(b, world * hp, s_loc, d)


def ulysses_attention(q_video: torch.Tensor, k_video: torch.Tensor, v_video: torch.Tensor,
                      q_text: torch.Tensor, k_text: torch.Tensor, v_text: torch.Tensor, *,
                      group=None, attn_fn: Callable | None = None, **kw):
    """Rectified sparse attention on sequence-sharded video tokens.

    q/k/v_video: [B, H, T_v/P, d] (this rank's contiguous slice of the video
    tokens); q/k/v_text: [B, H, T_t, d] replicated.  Returns
    (o_video [B, H, T_v/P, d], o_text [B, H, T_t, d] replicated)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    fn = attn_fn or _attention
    t_t = q_text.shape[2]
    h = q_video.shape[1]
    hp = h // world
    lo, hi = rank * hp, (rank + 1) * hp
    q = torch.cat([seq_to_head(q_video, group), q_text[:, lo:hi]], dim=2).contiguous()
    k = torch.cat([seq_to_head(k_video, group), k_text[:, lo:hi]], dim=2).contiguous()
    v = torch.cat([seq_to_head(v_video, group), v_text[:, lo:hi]], dim=2).contiguous()
    out = fn(q, k, v, t_t, **kw)                         # [B, H/P, T_v + T_t, d]
    t_v = out.shape[2] - t_t
    o_video = head_to_seq(out[:, :, :t_v].contiguous(), group)
    parts = [torch.empty_like(out[:, :, t_v:].contiguous()) for _ in range(world)]
    dist.all_gather(parts, out[:, :, t_v:].contiguous(), group=group)
    return o_video, torch.cat(parts, dim=1)
