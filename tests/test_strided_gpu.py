"""Strided Q/K/V/O views through rsa_forward_strided (include/rsa_b200.h): a
model's [B, T, H, d] projection output viewed as [B, H, T, d], and head
slices, run without any copy and give the contiguous call's bits.  The
reference's arrays are 2-D [T, d] (core.py:51-57); this is the batched form."""
import numpy as np
import pytest
import torch

import paper_2511_19835_b200 as rsa
from paper_2511_19835_b200 import _native as nat
from paper_2511_19835_b200.errors import NativeError

pytestmark = pytest.mark.gpu


def _inputs(B, H, T, d, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    # [B, T, H, d] storage, as a fused qkv projection leaves it
    return [torch.randn(B, T, H, d, generator=g).to(torch.bfloat16).cuda() for _ in range(3)]


def _rsa_kernels_only(fn):
    """Run fn under the profiler; return the names of the CUDA kernels it launched."""
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]


@pytest.mark.parametrize("d, block, t_v, t_t, kernel", [(128, 128, 128 * 24, 200, "tcgen05"),
                                                         (128, 128, 128 * 24, 200, "tcgen05-pingpong"),
                                                         (64, 64, 64 * 30, 100, "tcgen05")])
def test_bthd_view_equals_contiguous_bitwise(d, block, t_v, t_t, kernel):
    B, H = 2, 3
    qs, ks, vs = _inputs(B, H, t_v + t_t, d, 11)
    q, k, v = (x.transpose(1, 2) for x in (qs, ks, vs))          # [B, H, T, d] views, not contiguous
    assert not q.is_contiguous()
    kw = dict(num_text_tokens=t_t, block=block, top_k_fraction=0.2, weight_threshold=0.3, kernel=kernel)
    want = rsa.rectified_sparse_attention(q.contiguous(), k.contiguous(), v.contiguous(), **kw)
    lse = torch.empty(B * H * (t_v + t_t), dtype=torch.float32, device="cuda")
    got = rsa.rectified_sparse_attention(q, k, v, lse=lse, **kw)
    assert got.stride() == q.stride()                             # dense [B, T, H, d] storage, like q
    assert torch.equal(got, want)
    # the strided call launches the library's kernels and nothing of torch's
    # (no transpose / contiguous copy kernels; the status word's memset and
    # read-back are plain runtime calls)
    names = _rsa_kernels_only(lambda: rsa.rectified_sparse_attention(q, k, v, out=got, **kw))
    ours = [n for n in names if "rsa::" in n]
    others = [n for n in names if "rsa::" not in n and not n.startswith(("Memset", "Memcpy"))]
    assert ours and not others, others


def test_fused_qkv_slices_equal_contiguous_bitwise():
    """q/k/v as slices of one fused [B, T, 3, H, d] projection buffer (not
    dense: every token row skips the other two tensors); the output comes back
    as a dense [B, T, H, d] buffer viewed [B, H, T, d]."""
    B, H, T, d = 2, 2, 128 * 16 + 130, 128
    qkv = torch.randn(B, T, 3, H, d).to(torch.bfloat16).cuda()
    q, k, v = (qkv[:, :, i].transpose(1, 2) for i in range(3))
    kw = dict(num_text_tokens=130, block=128, top_k_fraction=0.25)
    want = rsa.rectified_sparse_attention(q.contiguous(), k.contiguous(), v.contiguous(), **kw)
    got = rsa.rectified_sparse_attention(q, k, v, **kw)
    assert got.transpose(1, 2).is_contiguous()
    assert torch.equal(got, want)
    # an explicit contiguous [B, H, T, d] out works too (its own layout)
    out = torch.empty(B, H, T, d, dtype=torch.bfloat16, device="cuda")
    rsa.rectified_sparse_attention(q, k, v, out=out, **kw)
    assert torch.equal(out, want)


def test_broadcast_kv_views_fall_back_to_copies():
    """k/v expanded over heads (stride 0, GQA-style) are not TMA-mappable views:
    the op copies them and still matches the materialised call."""
    B, H, T, d = 1, 3, 128 * 8 + 64, 128
    q = torch.randn(B, H, T, d).to(torch.bfloat16).cuda()
    k1, v1 = (torch.randn(B, 1, T, d).to(torch.bfloat16).cuda() for _ in range(2))
    k, v = k1.expand(B, H, T, d), v1.expand(B, H, T, d)
    kw = dict(num_text_tokens=64, block=128, top_k_fraction=0.3)
    want = rsa.rectified_sparse_attention(q, k.contiguous(), v.contiguous(), **kw)
    assert torch.equal(rsa.rectified_sparse_attention(q, k, v, **kw), want)


def test_strided_c_abi_rejects_unsupported_layouts():
    shape = nat.make_shape(2, 128 * 4, 0, 128, 128, "bfloat16")
    cfg = nat.make_config(0.5, 0.0, 0, False, "sparse-rectified")
    x = torch.zeros(2, 128 * 4, 128, dtype=torch.bfloat16, device="cuda")
    ws = torch.empty(nat.lib().rsa_workspace_size(shape), dtype=torch.uint8, device="cuda")
    p = lambda t: t.data_ptr()  # noqa: E731
    bad = nat.TensorLayout(2, 128 + 4, 128 * 4 * 128, 0)          # token stride not a multiple of 8
    with pytest.raises(NativeError):
        nat.check(nat.lib().rsa_forward_strided(shape, cfg, bad, None, p(x), p(x), p(x), p(x), None, p(ws), None))
    fp = nat.make_shape(2, 128 * 4, 0, 128, 128, "float32")
    y = torch.zeros(2, 128 * 4, 128, dtype=torch.float32, device="cuda")
    ok = nat.TensorLayout(2, 128, 128 * 4 * 128, 0)
    with pytest.raises(NativeError):                              # strided views are a bf16 / tcgen05 path
        nat.check(nat.lib().rsa_forward_strided(fp, cfg, ok, None, p(y), p(y), p(y), p(y), None, p(ws), None))
    bcast = nat.TensorLayout(2, 128, 0, 0)                         # a broadcast head dimension
    with pytest.raises(NativeError):
        nat.check(nat.lib().rsa_forward_strided(shape, cfg, bcast, None, p(x), p(x), p(x), p(x), None, p(ws), None))
