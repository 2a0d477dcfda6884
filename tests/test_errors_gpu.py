"""Error semantics of the model-facing entry points on the GPU.

The reference raises eagerly (core.py:23-31 non-finite -> ShapeError,
ipar.py:62-64 -> DegenerateRowError, kernel.py:85-87 -> EmptyRowError).  Here:
  * the batched op checks the device flags by default (one sync per call);
  * ``check_status=False`` + ``status=`` accumulates them on the stream;
  * the host-tensor call keeps the flags of every head chunk;
  * the C ABI's mask seam with an empty row returns RSA_ERR_EMPTY_ROW on the
    ping-pong tcgen05 kernel instead of hanging it;
  * caller workspaces / lse buffers are size-checked; mixed dtypes promote.
"""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2511_19835_b200 as rsa  # noqa: E402
from paper_2511_19835_b200 import _native as nat  # noqa: E402
from paper_2511_19835_b200.pipeline import _ptr, _stream, workspace_for  # noqa: E402
from oracle import rsa_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu


def qkv(heads, t_v, t_t, d, seed=0, device="cuda"):
    g = torch.Generator().manual_seed(seed)
    return [torch.randn(1, heads, t_v + t_t, d, generator=g).to(torch.bfloat16).to(device) for _ in range(3)]


def test_nan_in_late_head_of_host_call_raises():
    """rsa_forward_host runs K1-K3 per head chunk; a NaN in head 5 (chunk 5)
    must survive the later chunks' K1 and raise ShapeError."""
    q, k, v = qkv(8, 64 * 20, 64, 64, device="cpu")
    q[0, 5, 77, 3] = float("nan")
    with pytest.raises(rsa.ShapeError):
        rsa.rectified_sparse_attention(q.pin_memory(), k.pin_memory(), v.pin_memory(), num_text_tokens=64,
                                       block=64, sparsity=0.9, heads_per_chunk=1)
    q[0, 5, 77, 3] = 0.0
    out = rsa.rectified_sparse_attention(q.pin_memory(), k.pin_memory(), v.pin_memory(), num_text_tokens=64,
                                         block=64, sparsity=0.9, heads_per_chunk=1)
    assert torch.isfinite(out.float()).all()


def test_device_call_raises_by_default_and_accumulates_without_sync():
    q, k, v = qkv(3, 128 * 12, 100, 128)
    k[0, 2, 9, 1] = float("inf")
    with pytest.raises(rsa.ShapeError):
        rsa.rectified_sparse_attention(q, k, v, num_text_tokens=100, block=128, sparsity=0.9)
    status = rsa.new_status()
    good_k = k.clone()
    good_k[0, 2, 9, 1] = 0.0
    rsa.rectified_sparse_attention(q, good_k, v, num_text_tokens=100, block=128, sparsity=0.9,
                                   check_status=False, status=status)
    rsa.raise_for_status(status)          # nothing flagged yet
    rsa.rectified_sparse_attention(q, k, v, num_text_tokens=100, block=128, sparsity=0.9,
                                   check_status=False, status=status)
    rsa.rectified_sparse_attention(q, good_k, v, num_text_tokens=100, block=128, sparsity=0.9,
                                   check_status=False, status=status)
    with pytest.raises(rsa.ShapeError):   # sticky across the later clean call
        rsa.raise_for_status(status)


def test_torch_op_status_output():
    from paper_2511_19835_b200 import ops
    q, k, v = qkv(2, 64 * 10, 30, 64)
    v[0, 1, 3, 3] = float("nan")
    out, status = torch.ops.rsa_b200.rectified_sparse_attention_status(q, k, v, 30, 64, 0.1, 0.0, 0, False,
                                                                        "sparse-rectified")
    assert out.shape == q.shape
    with pytest.raises(rsa.ShapeError):
        rsa.raise_for_status(status)
    # the C++ operator raises RuntimeError naming the reference class; the
    # ops.py wrapper re-raises that class
    with pytest.raises(RuntimeError, match="^ShapeError: "):
        torch.ops.rsa_b200.rectified_sparse_attention(q, k, v, 30, 64, 0.1, 0.0, 0, False, "sparse-rectified")
    with pytest.raises(rsa.ShapeError):
        ops.rectified_sparse_attention(q, k, v, 30, 64, 0.1, 0.0, 0, False, "sparse-rectified")


@pytest.mark.timeout(180)
@pytest.mark.parametrize("kernel", ["tcgen05", "tcgen05-pingpong", "tcgen05-persistent"])
def test_empty_mask_rows_return_status_not_hang(kernel):
    """a video tile with an empty kv list issued no S MMA, so the
    ping-pong producer waited forever for its Q buffer.  The C ABI seam must
    return RSA_ERR_EMPTY_ROW on every d = B = 128 tcgen05 kernel -- with empty
    tiles in either slot of a pair, both slots of one pair, and CTAs that run
    further tiles after an empty one (64 heads: ~2 tile pairs per CTA) -- and
    the non-empty rows must equal the all-rows-retained call's rows."""
    heads, t_v, t_t, d, b = 64, 128 * 6, 0, 128, 128
    q, k, v = (x[0] for x in qkv(heads, t_v, t_t, d))
    shape = nat.make_shape(heads, t_v, t_t, d, b, "bfloat16", kernel)
    ws = workspace_for(shape, q.device)
    full = torch.ones(heads, 6, 6, dtype=torch.uint8, device="cuda")
    mask = full.clone()
    mask[0, 3] = 0            # slot 1 of a pair
    mask[0, 4] = mask[0, 5] = 0   # both slots of a pair
    mask[7, 0] = 0            # slot 0
    mask[40, 2] = 0
    lse = torch.empty(heads * (t_v + t_t), dtype=torch.float32, device="cuda")

    def run(m):
        out = torch.zeros_like(q)
        nat.check(nat.lib().rsa_block_sparse_attention(C.byref(shape), _ptr(q), _ptr(k), _ptr(v), _ptr(m),
                                                       _ptr(out), _ptr(lse), _ptr(ws), _stream()))
        return out, nat.lib().rsa_check_device_status(_ptr(ws), _stream())

    out, status = run(mask)
    assert status == 3   # RSA_ERR_EMPTY_ROW
    ref, status_ref = run(full)
    assert status_ref == 0
    torch.cuda.synchronize()
    keep = mask.bool().any(-1).repeat_interleave(b, dim=1)            # [heads, t_v] rows with a kv block
    assert torch.equal(out[keep], ref[keep])


def test_morton_check_status_without_workspace():
    """morton=True with check_status and no caller workspace."""
    grid = (2, 16, 16)
    q, k, v = qkv(2, 512, 64, 64)
    q[0, 1, 40, 0] = float("nan")
    with pytest.raises(rsa.ShapeError):
        rsa.rectified_sparse_attention(q, k, v, num_text_tokens=64, block=64, sparsity=0.8,
                                       grid_dims=grid, morton=True, check_status=True)
    q[0, 1, 40, 0] = 0.0
    out = rsa.rectified_sparse_attention(q, k, v, num_text_tokens=64, block=64, sparsity=0.8,
                                         grid_dims=grid, morton=True, check_status=True)
    assert torch.isfinite(out.float()).all()


def test_caller_workspace_and_lse_are_size_checked():
    q, k, v = qkv(2, 128 * 8, 16, 128)
    small = workspace_for(nat.make_shape(1, 128 * 8, 16, 128, 128, "bfloat16"), q.device)
    with pytest.raises(rsa.ShapeError):
        rsa.rectified_sparse_attention(q, k, v, num_text_tokens=16, block=128, sparsity=0.9, workspace=small)
    with pytest.raises(rsa.ShapeError):
        rsa.rectified_sparse_attention(q, k, v, num_text_tokens=16, block=128, sparsity=0.9,
                                       lse=torch.empty(10, device="cuda"))


def test_mixed_dtype_kernel_seams_promote_like_numpy():
    """q float32 with k/v float64 -> computed in float64 (numpy
    promotion in kernel.py), never read as the wrong element size."""
    qv, qt, k, v = O.random_problem(3, t_v=32, t_t=5, d=8, dtype=np.float64)
    n, m, last = O.block_geometry(32, 5, 8)
    mask = np.ones((n, m), dtype=bool)
    grid = rsa.partition(rsa.AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=8, block=8))
    out32, _ = rsa.block_sparse_attention(qv.astype(np.float32), k, v, mask, grid)
    out64, _ = rsa.block_sparse_attention(qv.astype(np.float32).astype(np.float64), k, v, mask, grid)
    assert out32.dtype == np.float64
    np.testing.assert_allclose(out32, out64, atol=1e-12, rtol=0)
    with pytest.raises(rsa.ShapeError):
        rsa.block_sparse_attention(qv, k[:-1], v[:-1], mask, grid)
    t32 = rsa.text_full_attention(qt.astype(np.float32), k, v, block=8)
    assert t32.dtype == np.float64
