"""CPU-side checks of the C++ TORCH_LIBRARY registration (csrc/torch_ops.cpp):
the schemas, the dispatch keys (CUDA + Meta, no CPU kernel), the Meta
kernels' output metadata (what torch.compile traces), and the host-side
validation raising the reference exception names.  No compute: the Meta
kernel only plans (rsa_plan)."""

import pytest
import torch

from paper_2511_19835_b200 import errors, ops

OP = "rsa_b200::rectified_sparse_attention"
OP_STATUS = "rsa_b200::rectified_sparse_attention_status"


def meta(*shape):
    return torch.empty(*shape, dtype=torch.bfloat16, device="meta")


def test_schemas_match_the_reference_argument_surface():
    # reference: core.py:51-57 (q/k/v, block), masks.py:30-33 (config), rectify.py:23-24 (variant)
    s = str(torch.ops.rsa_b200.rectified_sparse_attention.default._schema)
    for arg in ("Tensor q", "Tensor k", "Tensor v", "int num_text_tokens", "int block=128",
                "float top_k_fraction=0.1", "float weight_threshold=0.", "int adjacency_radius=0",
                "bool force_text_blocks=False", 'str variant="sparse-rectified"'):
        assert arg in s, (arg, s)
    assert s.endswith("-> Tensor")
    assert str(torch.ops.rsa_b200.rectified_sparse_attention_status.default._schema).endswith("-> (Tensor, Tensor)")


@pytest.mark.parametrize("name", [OP, OP_STATUS])
def test_registered_for_cuda_and_meta_only(name):
    has = torch._C._dispatch_has_kernel_for_dispatch_key
    assert has(name, "CUDA") and has(name, "Meta")
    assert not has(name, "CPU")
    q = torch.zeros(1, 2, 64 * 12 + 40, 64, dtype=torch.bfloat16)
    with pytest.raises(NotImplementedError):      # no CPU fallback
        torch.ops.rsa_b200.rectified_sparse_attention(q, q, q, 40, 64)


def test_meta_contiguous_output():
    q = meta(2, 3, 64 * 12 + 40, 64)
    out = torch.ops.rsa_b200.rectified_sparse_attention(q, q, q, 40, 64)
    assert out.shape == q.shape and out.is_contiguous() and out.dtype == torch.bfloat16
    out, status = torch.ops.rsa_b200.rectified_sparse_attention_status(q, q, q, 40, 64)
    assert out.shape == q.shape and status.shape == (4,) and status.dtype == torch.int32


def test_meta_strided_views_keep_the_model_layout():
    # [B, T, H, d] projection output viewed as [B, H, T, d]: the no-copy path,
    # output dense in q's dimension order
    x = meta(2, 128 * 7 + 64, 4, 128).transpose(1, 2)
    out = torch.ops.rsa_b200.rectified_sparse_attention(x, x, x, 64, 128)
    assert out.shape == x.shape and out.stride() == x.stride()
    # slices of a fused [B, T, 3, H, d] qkv buffer -> a dense [B, T, H, d] output
    qkv = meta(1, 64 * 10 + 30, 3, 2, 64)
    q, k, v = (qkv[:, :, i].transpose(1, 2) for i in range(3))
    out = torch.ops.rsa_b200.rectified_sparse_attention(q, k, v, 30, 64)
    assert out.shape == q.shape
    assert out.transpose(1, 2).is_contiguous()
    # a shape outside the tcgen05 kernels (d = 32) is copied: contiguous output
    y = meta(1, 64 * 4, 2, 32).transpose(1, 2)
    assert torch.ops.rsa_b200.rectified_sparse_attention(y, y, y, 0, 64).is_contiguous()
    # float32 always goes through the contiguous path
    z = torch.empty(1, 64 * 4, 2, 64, device="meta").transpose(1, 2)
    assert torch.ops.rsa_b200.rectified_sparse_attention(z, z, z, 0, 64).is_contiguous()


@pytest.mark.parametrize("args,cls", [
    ((41, 64), errors.BlockSizeError),                                     # core.py:71-72
    ((40, 64, 0.0), errors.ConfigError),                                   # masks.py:35-41
    ((40, 64, 0.1, 1.5), errors.ConfigError),
    ((40, 64, 0.1, 0.0, -1), errors.ConfigError),
    ((40, 64, 0.1, 0.0, 0, False, "bogus"), errors.ConfigError),          # rectify.py:118-119
])
def test_host_validation_names_the_reference_exception(args, cls):
    q = meta(1, 2, 64 * 12 + 40, 64)
    with pytest.raises(RuntimeError, match=f"^{cls.__name__}: "):
        torch.ops.rsa_b200.rectified_sparse_attention(q, q, q, *args)
    with pytest.raises(cls):
        ops.rectified_sparse_attention(q, q, q, *args)


def test_shape_and_dtype_errors():
    q = meta(1, 2, 64 * 12 + 40, 64)
    with pytest.raises(errors.ShapeError):
        ops.rectified_sparse_attention(q, meta(1, 2, 64 * 12 + 40, 32), q, 40, 64)
    with pytest.raises(errors.ShapeError):
        ops.rectified_sparse_attention(q, q.float(), q, 40, 64)
    with pytest.raises(errors.ShapeError):
        ops.rectified_sparse_attention(q.half(), q.half(), q.half(), 40, 64)
