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
    staged = dist.get_backend(group) != "nccl" and out.device.type != "cpu"   # gloo: host staging
    src = out.contiguous().cpu() if staged else out.contiguous()
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src, group=group)
    full = torch.cat(parts, dim=1)
    return full.to(out.device) if staged else full


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


def _a2a(recvs: list, sends: list, group, nccl: bool):
    """All-to-all of one head: ``sends[p]`` goes to rank p, rank p's piece
    lands in ``recvs[p]`` (contiguous [S/P, d] views, written in place).
    NCCL: list all-to-all (grouped ncclSend/ncclRecv, no staging copies),
    asynchronous on the process group's stream.  gloo (CPU tests, and the
    one-GPU plumbing run) only has the flat all_to_all_single: the sends are
    packed, CUDA tensors staged through host memory, synchronously."""
    if nccl:
        return dist.all_to_all(recvs, sends, group=group, async_op=True)
    packed = torch.stack(sends)
    packed = packed.cpu() if packed.device.type != "cpu" else packed
    got = torch.empty_like(packed)
    dist.all_to_all_single(got, packed, group=group)
    for p, r in enumerate(recvs):
        r.copy_(got[p])
    return None


def ulysses_attention(q_video: torch.Tensor, k_video: torch.Tensor, v_video: torch.Tensor,
                      q_text: torch.Tensor, k_text: torch.Tensor, v_text: torch.Tensor, *,
                      group=None, attn_fn: Callable | None = None, heads_per_group: int = 1, **kw):
    """Rectified sparse attention on sequence-sharded video tokens.

    q/k/v_video: [B, H, T_v/P, d] (this rank's contiguous slice of the video
    tokens); q/k/v_text: [B, H, T_t, d] replicated.  Returns
    (o_video [B, H, T_v/P, d], o_text [B, H, T_t, d] replicated).

    This rank's H/P heads run in groups of ``heads_per_group``: every input
    all-to-all is queued up front on the communication stream and group g's
    attention waits only for its own heads, so the shuffle of group g+1 (and
    the output shuffle of group g-1) overlaps group g's K1 -> K2 -> K3.  Each
    head's pieces are received straight into a preallocated [B, H/P, T, d]
    buffer whose text rows are filled once, and the attention writes into an
    output buffer the return shuffle reads in place -- no concatenation or
    permute copies (the send side reads strided per-head views)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    fn = attn_fn or _attention
    b, h, s_loc, d = q_video.shape
    if h % world:
        raise ValueError(f"heads ({h}) must be divisible by the world size ({world})")
    hp = h // world
    t_t = q_text.shape[2]
    t_v = s_loc * world
    T = t_v + t_t
    nccl = dist.get_backend(group) == "nccl"
    lo, hi = rank * hp, (rank + 1) * hp
    videos = (q_video, k_video, v_video)
    bufs = []
    for x, xt in zip(videos, (q_text, k_text, v_text)):
        buf = x.new_empty(b, hp, T, d)
        buf[:, :, t_v:] = xt[:, lo:hi]
        bufs.append(buf)
    groups = [(g0, min(hp, g0 + max(1, heads_per_group))) for g0 in range(0, hp, max(1, heads_per_group))]

    def shuffle_in(g0, g1):
        works = []
        for x, buf in zip(videos, bufs):
            for bi in range(b):
                for hl in range(g0, g1):
                    # rank p's slice of my head lo + hl -> rows [p S/P, (p+1) S/P) of my buffer
                    works.append(_a2a(list(buf[bi, hl, :t_v].chunk(world)),
                                      [x[bi, p * hp + hl] for p in range(world)], group, nccl))
        return [w for w in works if w is not None]

    pending = [shuffle_in(g0, g1) for g0, g1 in groups]
    obuf = q_video.new_empty(b, hp, T, d)
    o_video = q_video.new_empty(b, h, s_loc, d)
    out_works = []
    for (g0, g1), works in zip(groups, pending):
        for w in works:
            w.wait()                      # the compute stream waits for this group's heads only
        args = (bufs[0][:, g0:g1], bufs[1][:, g0:g1], bufs[2][:, g0:g1])
        if attn_fn is None and b == 1:
            fn(*args, t_t, out=obuf[:, g0:g1], **kw)
        else:
            obuf[:, g0:g1] = fn(*(a.contiguous() for a in args), t_t, **kw)
        for bi in range(b):
            for hl in range(g0, g1):
                # sequence slice p of my head lo + hl -> rank p; rank p's head p hp + hl -> my slice
                w = _a2a([o_video[bi, p * hp + hl] for p in range(world)],
                         list(obuf[bi, hl, :t_v].chunk(world)), group, nccl)
                if w is not None:
                    out_works.append(w)
    text = obuf[:, :, t_v:].contiguous()
    staged = not nccl and text.device.type != "cpu"   # gloo: host staging
    src = text.cpu() if staged else text
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src, group=group)
    o_text = torch.cat(parts, dim=1)
    for w in out_works:
        w.wait()
    return o_video, (o_text.to(text.device) if staged else o_text)
