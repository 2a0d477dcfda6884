"""Ragged final video block: an extension beyond
the reference, which raises BlockSizeError when T_v % B != 0 (core.py:71-72).
With ``ragged_video=True`` the last video block holds T_v - (N-1)B tokens:
it is pooled over its true length, stands for that many tokens in the IPAR
reallocation and in the GAPR gain/error, and K3 masks the missing rows and
keys.  Not parity-checkable against the reference; the oracle's extension
(oracle/rsa_oracle.py, ``ragged=True``) is pinned here by properties: it is
the reference path whenever T_v % B == 0, and its ``full`` variant equals dense
fp64 attention."""

import numpy as np
import pytest

from oracle import rsa_oracle as O
from paper_2511_19835_b200 import AttentionProblem, partition
from paper_2511_19835_b200 import _native as nat
from paper_2511_19835_b200.errors import BlockSizeError


# ----------------------------------------------------------------- CPU side

def test_default_still_raises_block_size_error():
    qv, qt, k, v = O.random_problem(0, t_v=37, t_t=5, d=8)
    with pytest.raises(BlockSizeError):
        AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=8, block=8)
    with pytest.raises(BlockSizeError):
        nat.plan(nat.make_shape(1, 37, 5, 8, 8, "float64"))
    with pytest.raises(O.OracleError):
        O.pipeline(qv, qt, k, v, 8)


def test_grid_of_a_ragged_problem():
    qv, qt, k, v = O.random_problem(0, t_v=37, t_t=5, d=8)
    prob = AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=8, block=8, ragged_video=True)
    grid = partition(prob)
    assert (grid.n_q, grid.n_kv, grid.last_video_block_len, grid.t_video) == (5, 6, 5, 37)
    assert grid.q_block_lengths() == [8, 8, 8, 8, 5]
    assert grid.kv_block_lengths() == [8, 8, 8, 8, 5, 5]
    g = nat.plan(nat.make_shape(1, 37, 5, 8, 8, "float64", ragged_video=True))
    assert (g.n_q, g.n_kv, g.last_video_block_len, g.last_text_block_len, g.n_cols) == (5, 6, 5, 5, 5 + 5 + 1)
    g = nat.plan(nat.make_shape(1, 40, 5, 8, 8, "float64", ragged_video=True))
    assert (g.n_q, g.last_video_block_len) == (5, 8)


def test_oracle_ragged_flag_is_the_reference_path_on_full_blocks():
    qv, qt, k, v = O.random_problem(3, t_v=48, t_t=10, d=8)
    a = O.pipeline(qv, qt, k, v, 8, 0.3, 0.3, 1, True)
    b = O.pipeline(qv, qt, k, v, 8, 0.3, 0.3, 1, True, ragged=True)
    for key in ("o_video", "o_text", "a_pool", "mask", "comp", "r", "gain", "error"):
        np.testing.assert_array_equal(a[key], b[key])


@pytest.mark.parametrize("t_v,t_t", [(37, 5), (33, 0), (9, 17)])
def test_oracle_ragged_full_variant_is_dense_attention(t_v, t_t):
    qv, qt, k, v = O.random_problem(1, t_v=t_v, t_t=t_t, d=8)
    res = O.pipeline(qv, qt, k, v, 8, variant="full", ragged=True)
    _, dense = O.full_attention_fp64(np.concatenate([qv, qt]), k, v)
    np.testing.assert_allclose(res["o_video"], dense[:t_v], atol=1e-12, rtol=0)
    np.testing.assert_allclose(res["o_text"], dense[t_v:], atol=1e-12, rtol=0)
    assert np.all(res["r"] == 1.0)
    # the ragged block is pooled over its true length and stands for that many tokens
    pooled = res["pooled"]
    np.testing.assert_allclose(pooled["q_pool"][-1], qv[(res["n_q"] - 1) * 8:].mean(axis=0), atol=1e-15)
    assert pooled["q_lens"][-1] == t_v - (res["n_q"] - 1) * 8
    # IPAR rows stay distributions
    np.testing.assert_allclose(res["a_pool"].sum(axis=1), 1.0, atol=1e-12)


# ----------------------------------------------------------------- GPU parity

torch = pytest.importorskip("torch")
rsa = pytest.importorskip("paper_2511_19835_b200")
from paper_2511_19835_b200 import SparsityConfig  # noqa: E402


def _run(qv, qt, k, v, block, cfg, variant, kernel="auto"):
    prob = AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=qv.shape[1], block=block, ragged_video=True)
    return rsa.rectified_attention_pipeline(prob, SparsityConfig(*cfg), variant, kernel=kernel)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-12), (np.float32, 1e-5)])
@pytest.mark.parametrize("t_v,t_t,block", [(37, 5, 8), (33, 0, 8), (70, 13, 16), (9, 17, 8)])
def test_gpu_ragged_small_vs_oracle(dtype, tol, t_v, t_t, block):
    qv, qt, k, v = O.random_problem(5, t_v=t_v, t_t=t_t, d=8, dtype=dtype)
    cfg = (0.4, 0.3, 1, True)
    for variant in O.VARIANTS:
        res = _run(qv, qt, k, v, block, cfg, variant)
        ref = O.pipeline(qv, qt, k, v, block, *cfg, variant=variant, ragged=True)
        np.testing.assert_array_equal(res.sparse_mask.mask, ref["mask"])
        np.testing.assert_array_equal(res.comp_mask.mask, ref["comp"])
        np.testing.assert_allclose(res.implicit.a_pool, ref["a_pool"], atol=1e-12, rtol=0)
        np.testing.assert_allclose(res.factors.r, ref["r"], atol=1e-12, rtol=0)
        np.testing.assert_allclose(res.output.o_video, ref["o_video"], atol=tol, rtol=0)
        np.testing.assert_allclose(res.output.o_text, ref["o_text"], atol=tol, rtol=0)


def _bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).cuda()


@pytest.mark.gpu
@pytest.mark.parametrize("block,d,t_v,t_t", [(64, 64, 64 * 60 - 23, 256), (128, 128, 128 * 20 + 16, 200),
                                             (128, 128, 128 * 21 - 1, 0), (64, 128, 64 * 30 + 5, 129)])
def test_gpu_ragged_tcgen05_vs_oracle(block, d, t_v, t_t):
    """bf16 tensor-core path: masks / gate bit-exact, outputs within the bf16 bar."""
    qv, qt, k, v = (O.round_to_bf16(x) for x in O.random_problem(11, t_v=t_v, t_t=t_t, d=d, dtype=np.float32))
    cfg = (0.1, 0.0, 0, False)
    prob = AttentionProblem(q_video=_bf16(qv), q_text=_bf16(qt), k=_bf16(k), v=_bf16(v), d=d, block=block,
                            ragged_video=True)
    for variant in ("sparse-rectified", "full"):
        res = rsa.rectified_attention_pipeline(prob, SparsityConfig(*cfg), variant)
        ref = O.pipeline(qv, qt, k, v, block, *cfg, variant=variant, ragged=True)
        np.testing.assert_array_equal(res.sparse_mask.mask.cpu().numpy(), ref["mask"])
        np.testing.assert_array_equal(res.comp_mask.mask.cpu().numpy(), ref["comp"])
        for got, want in ((res.output.o_video, ref["o_video"]), (res.output.o_text, ref["o_text"])):
            if want.shape[0] == 0:
                continue
            got = got.float().cpu().numpy().astype(np.float64)
            assert np.abs(got - want).max() <= 2e-2
            assert O.cosine(got, want) >= 0.999


@pytest.mark.gpu
def test_gpu_ragged_hunyuan_exact_token_count():
    """HunyuanVideo's exact 118,800 video tokens (928 full blocks + 16): the
    batched op with ragged_video=True; head 0's mask bit-exact against the
    oracle's pooled path, every output finite."""
    t_v, t_t, d, block = 118800, 256, 128, 128
    qv, qt, k, v = O.gen_synthetic(42, 118784, t_t, d, block, (29, 64, 64), 1.0, 2.0, 0.3)
    rng = np.random.default_rng(0)
    extra = [rng.standard_normal((16, d)).astype(np.float32) for _ in range(3)]
    qv = np.concatenate([qv, extra[0]])
    k = np.concatenate([k[:118784], extra[1], k[118784:]])
    v = np.concatenate([v[:118784], extra[2], v[118784:]])
    qv, qt, k, v = (O.round_to_bf16(x) for x in (qv, qt, k, v))
    q = torch.cat([_bf16(qv), _bf16(qt)])[None, None]
    out = rsa.rectified_sparse_attention(q, _bf16(k)[None, None], _bf16(v)[None, None], num_text_tokens=t_t,
                                         block=block, sparsity=0.9, ragged_video=True, check_status=True)
    assert out.shape == q.shape and bool(torch.isfinite(out.float()).all())
    prob = AttentionProblem(q_video=_bf16(qv), q_text=_bf16(qt), k=_bf16(k), v=_bf16(v), d=d, block=block,
                            ragged_video=True)
    res = rsa.rectified_attention_pipeline(prob, SparsityConfig(0.1, 0.0, 0, False))
    pooled = O.pool(qv, k, v, t_t, block, ragged=True)
    imp = O.implicit_attention(pooled, d, block, t_t)
    sel = O.select_mask(imp["a_pool"], 0.1, 0.0, 0, False, pooled["n_q"])
    np.testing.assert_array_equal(res.sparse_mask.mask.cpu().numpy(), sel["mask"])
    np.testing.assert_allclose(res.implicit.a_pool.cpu().numpy(), imp["a_pool"], atol=1e-12, rtol=0)
    assert torch.equal(res.output.o_video, out[0, 0, :t_v])


@pytest.mark.gpu
def test_gpu_ragged_fused_morton_matches_oracle():
    """Ragged final video block + fused Morton reorder (K1 gather, K3 scatter):
    the reordered problem's masks bit-exact against the oracle's extension,
    outputs back in the original token order within the bf16 bar."""
    from paper_2511_19835_b200.pipeline import workspace_for
    grid, block, d, t_t = (3, 10, 9), 64, 64, 70
    t_v = grid[0] * grid[1] * grid[2]                # 270 = 4 * 64 + 14
    qv, qt, k, v = (O.round_to_bf16(x) for x in O.random_problem(21, t_v=t_v, t_t=t_t, d=d, dtype=np.float32))
    q = torch.cat([_bf16(qv), _bf16(qt)])[None]
    shape = nat.make_shape(1, t_v, t_t, d, block, "bfloat16", ragged_video=True)
    ws = workspace_for(shape, "cuda")
    out = rsa.rectified_sparse_attention(q, _bf16(k)[None], _bf16(v)[None], num_text_tokens=t_t, block=block,
                                         top_k_fraction=0.4, grid_dims=grid, morton=True, workspace=ws,
                                         check_status=True, ragged_video=True)[0]
    rq, rqt, rk, rv, perm = O.reorder_morton(qv, qt, k, v, grid)
    ref = O.pipeline(rq, rqt, rk, rv, block, 0.4, 0.0, 0, False, "sparse-rectified", ragged=True)
    L = nat.layout(shape)
    n, m = ref["mask"].shape
    bits = ws[L["mask_bits"]:L["mask_bits"] + n * m].view(n, m).cpu().numpy()
    np.testing.assert_array_equal((bits & 1) != 0, ref["mask"])
    want = np.empty((t_v + t_t, d), np.float64)
    want[perm] = ref["o_video"]
    want[t_v:] = ref["o_text"]
    got = out.float().cpu().numpy().astype(np.float64)
    assert np.abs(got - want).max() <= 2e-2 and O.cosine(got, want) >= 0.999
