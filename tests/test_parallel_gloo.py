"""Multi-process (world_size 2, gloo, CPU) tests of the head-sharding and
Ulysses all-to-all plumbing.  The attention callable is the CPU oracle here
(the CUDA op runs the same data movement on the GPU box)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rsa_oracle as O
from paper_2511_19835_b200.parallel import (head_parallel_attention, head_range, head_to_seq,
                                            seq_to_head, ulysses_attention)

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def oracle_attn(q, k, v, num_text_tokens, block=8, top_k_fraction=0.3):
    """Per-(batch, head) oracle pipeline on [B, H, T, d] tensors."""
    out = torch.empty_like(q)
    t_v = q.shape[2] - num_text_tokens
    for b in range(q.shape[0]):
        for h in range(q.shape[1]):
            qq, kk, vv = (x[b, h].numpy() for x in (q, k, v))
            r = O.pipeline(qq[:t_v], qq[t_v:], kk, vv, block, top_k_fraction, 0.0, 0, False,
                           "sparse-rectified")
            out[b, h] = torch.from_numpy(np.concatenate([r["o_video"], r["o_text"]]))
    return out


def _problem(seed=0, b=1, h=4, t_v=64, t_t=5, d=8):
    g = torch.Generator().manual_seed(seed)
    mk = lambda t: torch.randn(b, h, t, d, generator=g, dtype=torch.float64)  # noqa: E731
    return mk(t_v), mk(t_t), mk(t_v), mk(t_t), mk(t_v), mk(t_t)


def _worker(rank, port, fn_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        globals()[fn_name](rank, q)
    except Exception as exc:  # report to the parent
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()
    q.put((rank, "ok"))


def _run(fn_name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, fn_name, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    results = [q.get(timeout=5) for _ in range(WORLD)]
    assert all(msg == "ok" for _, msg in results), results


def check_shuffle_roundtrip(rank, _q):
    qv, *_ = _problem()
    s_loc = qv.shape[2] // WORLD
    mine = qv[:, :, rank * s_loc:(rank + 1) * s_loc].contiguous()
    heads = seq_to_head(mine)
    hp = qv.shape[1] // WORLD
    torch.testing.assert_close(heads, qv[:, rank * hp:(rank + 1) * hp], rtol=0, atol=0)
    torch.testing.assert_close(head_to_seq(heads), mine, rtol=0, atol=0)


def check_ulysses_matches_single_process(rank, _q):
    qv, qt, kv, kt, vv, vt = _problem(seed=3)
    s_loc = qv.shape[2] // WORLD
    sl = slice(rank * s_loc, (rank + 1) * s_loc)
    o_video, o_text = ulysses_attention(qv[:, :, sl].contiguous(), kv[:, :, sl].contiguous(),
                                        vv[:, :, sl].contiguous(), qt, kt, vt, attn_fn=oracle_attn)
    full = oracle_attn(torch.cat([qv, qt], 2), torch.cat([kv, kt], 2), torch.cat([vv, vt], 2), qt.shape[2])
    torch.testing.assert_close(o_video, full[:, :, :qv.shape[2]][:, :, sl], rtol=0, atol=0)
    torch.testing.assert_close(o_text, full[:, :, qv.shape[2]:], rtol=0, atol=0)


def check_ulysses_grouped_batched(rank, _q):
    """Two batch entries, head groups of 2 (each group's shuffle overlaps the
    previous group's attention on NCCL; here the same data movement, gloo)."""
    qv, qt, kv, kt, vv, vt = _problem(seed=4, b=2, h=4)
    s_loc = qv.shape[2] // WORLD
    sl = slice(rank * s_loc, (rank + 1) * s_loc)
    for hpg in (1, 2):
        o_video, o_text = ulysses_attention(qv[:, :, sl].contiguous(), kv[:, :, sl].contiguous(),
                                            vv[:, :, sl].contiguous(), qt, kt, vt, attn_fn=oracle_attn,
                                            heads_per_group=hpg)
        full = oracle_attn(torch.cat([qv, qt], 2), torch.cat([kv, kt], 2), torch.cat([vv, vt], 2), qt.shape[2])
        torch.testing.assert_close(o_video, full[:, :, :qv.shape[2]][:, :, sl], rtol=0, atol=0)
        torch.testing.assert_close(o_text, full[:, :, qv.shape[2]:], rtol=0, atol=0)


def check_head_parallel_gather(rank, _q):
    qv, qt, kv, kt, vv, vt = _problem(seed=5)
    q, k, v = torch.cat([qv, qt], 2), torch.cat([kv, kt], 2), torch.cat([vv, vt], 2)
    out = head_parallel_attention(q, k, v, num_text_tokens=qt.shape[2], gather=True, attn_fn=oracle_attn)
    torch.testing.assert_close(out, oracle_attn(q, k, v, qt.shape[2]), rtol=0, atol=0)


def test_head_range_balanced():
    assert [head_range(24, 8, r) for r in range(8)] == [(3 * r, 3 * r + 3) for r in range(8)]
    spans = [head_range(40, 3, r) for r in range(3)]
    assert spans == [(0, 14), (14, 27), (27, 40)]


@pytest.mark.parametrize("fn", ["check_shuffle_roundtrip", "check_ulysses_matches_single_process",
                                "check_ulysses_grouped_batched", "check_head_parallel_gather"])
def test_gloo_world2(fn):
    _run(fn)
