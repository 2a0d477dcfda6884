"""GPU parity: the sm_100a pipeline (through the C ABI) against the CPU oracle
and the reference goldens.  Bars (BASELINE.json):
  * block masks / importance / gain>error gate: bit-exact
  * a_pool, R: <= 1e-12 abs; pooled tensors bit-exact
  * fp64 inputs: outputs <= 1e-12; fp32 inputs: <= 1e-5 (reference tolerances,
    pkg/tests/test_kernel.py:62-77)
  * bf16 inputs (tensor-core path): max-abs <= 2e-2 and cosine >= 0.999 vs the
    fp32 oracle pipeline on the same bf16-valued inputs.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2511_19835_b200 as rsa  # noqa: E402
from paper_2511_19835_b200 import AttentionProblem, SparsityConfig, partition  # noqa: E402
from conftest import N_TINY, tiny_case  # noqa: E402
from oracle import rsa_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

BF16_MAX_ABS = 2e-2
BF16_MIN_COS = 0.999


def to_bf16_tensor(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).cuda()


def run_np(qv, qt, k, v, block, f, p, r, force, variant, kernel="auto"):
    prob = AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=qv.shape[1], block=block)
    return rsa.rectified_attention_pipeline(prob, SparsityConfig(f, p, r, force), variant, kernel=kernel)


# ---------------------------------------------------------------- tiny goldens

@pytest.mark.parametrize("i", range(N_TINY))
def test_tiny_cases_against_reference_goldens(tiny_golden, i):
    (qv, qt, k, v), m = tiny_case(tiny_golden, i)
    tol = 1e-12 if qv.dtype == np.float64 else 1e-5
    for variant in O.VARIANTS:
        res = run_np(qv, qt, k, v, m["block"], m["f"], m["p"], m["r"], m["force"], variant)
        tag = f"c{i}_{variant}"
        assert res.output.o_video.dtype == qv.dtype
        np.testing.assert_allclose(res.output.o_video, tiny_golden[f"{tag}_o_video"], atol=tol, rtol=0)
        np.testing.assert_allclose(res.output.o_text, tiny_golden[f"{tag}_o_text"], atol=tol, rtol=0)
        if variant == "sparse-rectified":
            np.testing.assert_array_equal(res.sparse_mask.mask, tiny_golden[f"c{i}_mask"])
            np.testing.assert_array_equal(res.sparse_mask.importance, tiny_golden[f"c{i}_importance"])
            np.testing.assert_array_equal(res.comp_mask.mask, tiny_golden[f"c{i}_comp"])
            np.testing.assert_allclose(res.factors.r, tiny_golden[f"c{i}_r"], atol=1e-12, rtol=0)
            np.testing.assert_allclose(res.implicit.a_pool, tiny_golden[f"c{i}_a_pool"], atol=1e-12, rtol=0)
            np.testing.assert_array_equal(res.pooled.q_pool, tiny_golden[f"c{i}_q_pool"])
            np.testing.assert_array_equal(res.pooled.v_pool, tiny_golden[f"c{i}_v_pool"])
            np.testing.assert_array_equal(res.pooled.k_mix_pool, tiny_golden[f"c{i}_k_mix"])
            assert rsa.check_result_invariants(res)


# ---------------------------------------------------------------- cfg1 (bf16)

def cfg1_inputs(seed):
    qv, qt, k, v = O.gen_synthetic(seed, 3840, 256, 64, 64, (1, 60, 64), 1.0, 2.0, 0.3)
    return tuple(O.round_to_bf16(x) for x in (qv, qt, k, v))


def bf16_problem(qv, qt, k, v, block):
    return AttentionProblem(q_video=to_bf16_tensor(qv), q_text=to_bf16_tensor(qt),
                            k=to_bf16_tensor(k), v=to_bf16_tensor(v), d=qv.shape[1], block=block)


def assert_bf16_close(got, ref, what):
    got = got.float().cpu().numpy().astype(np.float64) if torch.is_tensor(got) else np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(got - ref).max()
    cos = O.cosine(got, ref)
    assert err <= BF16_MAX_ABS and cos >= BF16_MIN_COS, f"{what}: max-abs {err:.3e}, cos {cos:.6f}"


@pytest.mark.parametrize("seed", [42, 43])
@pytest.mark.parametrize("kernel", ["auto", "simt"])
def test_cfg1_bf16_masks_bit_exact_and_outputs(cfg1_golden, seed, kernel):
    qv, qt, k, v = cfg1_inputs(seed)
    prob = bf16_problem(qv, qt, k, v, 64)
    for f in (0.5, 0.25, 0.1, 0.05):
        for p in (0.0, 0.5):
            res = rsa.rectified_attention_pipeline(prob, SparsityConfig(f, p, 0, False),
                                                   "sparse-rectified", kernel=kernel)
            mask = res.sparse_mask.mask.cpu().numpy()
            np.testing.assert_array_equal(np.packbits(mask, axis=1), cfg1_golden[f"s{seed}_f{f}_p{p}_mask"])
            np.testing.assert_allclose(res.factors.r.cpu().numpy(), cfg1_golden[f"s{seed}_f{f}_p{p}_r"],
                                       atol=1e-12, rtol=0)
            np.testing.assert_array_equal(np.packbits(res.comp_mask.mask.cpu().numpy(), axis=1),
                                          cfg1_golden[f"s{seed}_comp"])
            assert_bf16_close(res.output.o_video[::32], cfg1_golden[f"s{seed}_f{f}_p{p}_sparse-rectified_o_rows"],
                              f"f={f} p={p} video")
            assert_bf16_close(res.output.o_text[::8], cfg1_golden[f"s{seed}_f{f}_p{p}_sparse-rectified_ot_rows"],
                              f"f={f} p={p} text")
    np.testing.assert_allclose(res.implicit.a_pool.cpu().numpy(), cfg1_golden[f"s{seed}_a_pool"],
                               atol=1e-12, rtol=0)


@pytest.mark.parametrize("variant", O.VARIANTS)
def test_cfg1_bf16_all_variants_full_output_vs_oracle(variant):
    qv, qt, k, v = cfg1_inputs(42)
    res = rsa.rectified_attention_pipeline(bf16_problem(qv, qt, k, v, 64),
                                           SparsityConfig(0.1, 0.0, 0, False), variant)
    ref = O.pipeline(qv, qt, k, v, 64, 0.1, 0.0, 0, False, variant)
    np.testing.assert_array_equal(res.sparse_mask.mask.cpu().numpy(), ref["mask"])
    assert_bf16_close(res.output.o_video, ref["o_video"], f"{variant} video")
    assert_bf16_close(res.output.o_text, ref["o_text"], f"{variant} text")


def test_batched_tensor_op_matches_per_head_oracle():
    heads = [cfg1_inputs(s) for s in (42, 43)]
    q = torch.stack([torch.cat([to_bf16_tensor(h[0]), to_bf16_tensor(h[1])]) for h in heads])[None]
    k = torch.stack([to_bf16_tensor(h[2]) for h in heads])[None]
    v = torch.stack([to_bf16_tensor(h[3]) for h in heads])[None]
    out = rsa.rectified_sparse_attention(q, k, v, num_text_tokens=256, block=64, sparsity=0.9,
                                         check_status=True)
    assert out.shape == q.shape and out.dtype == torch.bfloat16
    for i, (qv, qt, kk, vv) in enumerate(heads):
        ref = O.pipeline(qv, qt, kk, vv, 64, 1.0 - 0.9, 0.0, 0, False, "sparse-rectified")
        assert_bf16_close(out[0, i], np.concatenate([ref["o_video"], ref["o_text"]]), f"head {i}")


def test_torch_library_op():
    from paper_2511_19835_b200 import ops  # noqa: F401  (registers torch.ops.rsa_b200)
    qv, qt, k, v = cfg1_inputs(42)
    q = torch.cat([to_bf16_tensor(qv), to_bf16_tensor(qt)])[None]
    out = torch.ops.rsa_b200.rectified_sparse_attention(q, to_bf16_tensor(k)[None], to_bf16_tensor(v)[None],
                                                        256, 64, 0.1, 0.0, 0, False, "sparse-rectified")
    ref = O.pipeline(qv, qt, k, v, 64, 0.1, 0.0, 0, False, "sparse-rectified")
    assert_bf16_close(out[0], np.concatenate([ref["o_video"], ref["o_text"]]), "torch.ops")


def test_torch_library_op_equals_the_c_abi_call():
    """The C++ TORCH_LIBRARY op (csrc/torch_ops.cpp) and the ctypes C-ABI API
    run the same kernels: bitwise equal outputs, contiguous and through the
    no-copy strided path (a [B, T, H, d] view and fused-qkv slices)."""
    from paper_2511_19835_b200 import ops  # noqa: F401
    g = torch.Generator().manual_seed(5)
    qkv = torch.randn(1, 128 * 9 + 64, 3, 4, 128, generator=g).to(torch.bfloat16).cuda()
    q, k, v = (qkv[:, :, i].transpose(1, 2) for i in range(3))
    kw = dict(num_text_tokens=64, block=128, top_k_fraction=0.25, weight_threshold=0.0, adjacency_radius=1,
              force_text_blocks=True, variant="sparse-rectified")
    want = rsa.rectified_sparse_attention(q.contiguous(), k.contiguous(), v.contiguous(), **kw)
    for args in ((q, k, v), (q.contiguous(), k.contiguous(), v.contiguous())):
        got = torch.ops.rsa_b200.rectified_sparse_attention(*args, *kw.values())
        assert torch.equal(got, want)
        got, status = torch.ops.rsa_b200.rectified_sparse_attention_status(*args, *kw.values())
        assert torch.equal(got, want)
        rsa.raise_for_status(status)


def test_torch_library_op_fp32_and_small_head_dim():
    """The C++ op on the other shape classes: fp32 (CUDA-core K3, contiguous
    copy of a strided input) against the fp64 oracle, and a d = B = 64 bf16
    [B, T, H, d] view (persistent tcgen05 K3, no-copy path) against the
    contiguous call, bitwise."""
    from paper_2511_19835_b200 import ops  # noqa: F401
    qv, qt, k, v = O.gen_synthetic(7, 64 * 12, 40, 64, 64, (1, 12, 64), 1.0, 2.0, 0.3)
    q32 = torch.from_numpy(np.concatenate([qv, qt]).astype(np.float32)).cuda()[None]
    k32 = torch.from_numpy(k.astype(np.float32)).cuda()[None]
    v32 = torch.from_numpy(v.astype(np.float32)).cuda()[None]
    out = torch.ops.rsa_b200.rectified_sparse_attention(q32, k32, v32, 40, 64, 0.25, 0.0, 0, False,
                                                        "sparse-rectified")
    ref = O.pipeline(qv.astype(np.float64), qt.astype(np.float64), k.astype(np.float64), v.astype(np.float64),
                     64, 0.25, 0.0, 0, False, "sparse-rectified")
    np.testing.assert_allclose(out[0].cpu().numpy(), np.concatenate([ref["o_video"], ref["o_text"]]),
                               atol=1e-5, rtol=0)
    g = torch.Generator().manual_seed(9)
    x = [torch.randn(2, 64 * 10 + 30, 3, 64, generator=g).to(torch.bfloat16).cuda() for _ in range(3)]
    qs, ks, vs = (t.transpose(1, 2) for t in x)          # [B, H, T, d] views
    got = torch.ops.rsa_b200.rectified_sparse_attention(qs, ks, vs, 30, 64, 0.2, 0.0, 0, False, "sparse-rectified")
    want = torch.ops.rsa_b200.rectified_sparse_attention(qs.contiguous(), ks.contiguous(), vs.contiguous(), 30, 64,
                                                         0.2, 0.0, 0, False, "sparse-rectified")
    assert got.stride() == qs.stride() and torch.equal(got, want)


def test_torch_library_opcheck_and_compile():
    """torch.library.opcheck (schema, fake/meta kernel vs the CUDA kernel,
    AOT dispatch) on the registered op, contiguous and strided inputs, and a
    torch.compile(fullgraph=True) graph that calls it."""
    from paper_2511_19835_b200 import ops  # noqa: F401
    op = torch.ops.rsa_b200.rectified_sparse_attention.default
    g = torch.Generator().manual_seed(3)
    x = [torch.randn(1, 64 * 12 + 40, 2, 64, generator=g).to(torch.bfloat16).cuda() for _ in range(3)]
    args = (40, 64, 0.3, 0.2, 1, True, "sparse-rectified")
    for q, k, v in (tuple(t.transpose(1, 2).contiguous() for t in x), tuple(t.transpose(1, 2) for t in x)):
        torch.library.opcheck(op, (q, k, v) + args)

    def f(q, k, v):
        return torch.ops.rsa_b200.rectified_sparse_attention(q, k, v, *args) * 0.5

    q, k, v = (t.transpose(1, 2) for t in x)
    compiled = torch.compile(f, fullgraph=True, backend="aot_eager")
    assert torch.equal(compiled(q, k, v), f(q, k, v))


def test_determinism_bitwise():
    qv, qt, k, v = cfg1_inputs(43)
    prob = bf16_problem(qv, qt, k, v, 64)
    a = rsa.rectified_attention_pipeline(prob, SparsityConfig(0.1, 0.0, 0, False))
    b = rsa.rectified_attention_pipeline(prob, SparsityConfig(0.1, 0.0, 0, False))
    assert torch.equal(a.output.o_video, b.output.o_video)
    assert torch.equal(a.output.o_text, b.output.o_text)


# ---------------------------------------------------------------- full-size masks

def test_hunyuan_head_mask_bit_exact(large_golden):
    """HunyuanVideo 720p head (T_v=118,784, T_t=256, d=128, B=128): the whole
    pooled path on the GPU reproduces the reference mask bit-for-bit."""
    qv, qt, k, v = O.gen_synthetic(42, 118784, 256, 128, 128, (29, 64, 64), 1.0, 2.0, 0.3)
    qv, qt, k, v = (O.round_to_bf16(x) for x in (qv, qt, k, v))
    prob = bf16_problem(qv, qt, k, v, 128)
    for f in (0.1, 0.05):
        res = rsa.rectified_attention_pipeline(prob, SparsityConfig(f, 0.0, 0, False))
        mask = res.sparse_mask.mask.cpu().numpy()
        np.testing.assert_array_equal(np.packbits(mask, axis=1), large_golden[f"hv_s42_f{f}_mask"])
        np.testing.assert_allclose(res.factors.r.cpu().numpy(), large_golden[f"hv_s42_f{f}_r"],
                                   atol=1e-12, rtol=0)
        sp = 1.0 - mask.sum() / mask.size
        assert 0.85 < sp < 0.96
    # size-independent property at full size: every output row is finite and
    # R in (0, 1]
    assert torch.isfinite(res.output.o_video.float()).all()
    assert (res.factors.r > 0).all() and (res.factors.r <= 1 + 1e-12).all()


def test_wan_head_mask_bit_exact(large_golden):
    rng = np.random.default_rng(42)
    t = 75520
    qv = O.round_to_bf16(rng.standard_normal((t, 128)).astype(np.float32))
    k = O.round_to_bf16(rng.standard_normal((t, 128)).astype(np.float32))
    v = O.round_to_bf16(rng.standard_normal((t, 128)).astype(np.float32))
    qt = np.zeros((0, 128), dtype=np.float32)
    res = rsa.rectified_attention_pipeline(bf16_problem(qv, qt, k, v, 128), SparsityConfig(0.1, 0.0, 0, False))
    mask = res.sparse_mask.mask.cpu().numpy()
    np.testing.assert_array_equal(np.packbits(mask, axis=1), large_golden["wan_s42_f0.1_mask"])
    np.testing.assert_allclose(res.factors.r.cpu().numpy(), large_golden["wan_s42_f0.1_r"], atol=1e-12, rtol=0)


# ---------------------------------------------------------------- kernel seams

@pytest.mark.parametrize("precision,tol", [("single", 1e-5), ("double", 1e-12)])
def test_block_sparse_attention_random_masks(precision, tol):
    """pkg/tests/test_kernel.py:62-77 on the GPU kernel."""
    rng = np.random.default_rng(7)
    dtype = np.float32 if precision == "single" else np.float64
    for i in range(20):
        block = int(rng.choice([4, 8, 16]))
        t_v = block * int(rng.integers(2, 9))
        t_t = int(rng.integers(0, 9))
        d = int(rng.choice([8, 16]))
        qv, qt, k, v = O.random_problem(100 + i, t_v=t_v, t_t=t_t, d=d, dtype=dtype)
        n, m, last = O.block_geometry(t_v, t_t, block)
        lens = O.kv_lengths(n, m, block, last)
        mask = rng.random((n, m)) < 0.4
        for row in range(n):
            if not mask[row].any():
                mask[row, rng.integers(0, m)] = True
        grid = partition(AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=d, block=block))
        counters = {}
        out, ld = rsa.block_sparse_attention(qv, k, v, mask, grid, counters=counters)
        _, expected = O.masked_attention_fp64(qv, k, v, mask, lens, block)
        assert np.abs(out.astype(np.float64) - expected).max() <= tol
        assert counters["inner_product_ops"] == int((mask * np.asarray(lens)[None, :]).sum()) * block * d
        assert ld.shape == (t_v,)


def test_block_sparse_attention_empty_row_rejected():
    qv, qt, k, v = O.random_problem(2, t_v=8, t_t=0, d=8)
    grid = partition(AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=8, block=4))
    mask = np.zeros((2, 2), dtype=bool)
    mask[0, 0] = True
    with pytest.raises(rsa.EmptyRowError):
        rsa.block_sparse_attention(qv, k, v, mask, grid)


@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-5), (np.float64, 1e-12)])
def test_text_full_attention(dtype, tol):
    qv, qt, k, v = O.random_problem(9, t_v=32, t_t=11, d=8, dtype=dtype)
    out = rsa.text_full_attention(qt, k, v, block=4)
    _, expected = O.full_attention_fp64(qt, k, v)
    assert np.abs(out.astype(np.float64) - expected).max() <= tol
    assert rsa.text_full_attention(qt[:0], k, v, block=4).shape == (0, 8)


def test_uniform_rows_tie_break_on_gpu():
    """Identical keys -> uniform a_pool rows; ties resolve to ascending block
    index (pkg/tests/test_masks.py:38-49)."""
    rng = np.random.default_rng(3)
    d, block, t_v = 8, 4, 32
    qv = rng.standard_normal((t_v, d))
    k = np.tile(rng.standard_normal((1, d)), (t_v, 1))
    v = rng.standard_normal((t_v, d))
    res = run_np(qv, np.zeros((0, d)), k, v, block, 0.25, 0.0, 1, False, "sparse-rectified")
    for n in range(8):
        adj = {m for m in (n - 1, n, n + 1) if 0 <= m < 8}
        assert set(np.flatnonzero(res.sparse_mask.mask[n])) == adj | {0, 1}


def test_zero_sparsity_identity_fp32():
    """pkg/tests/test_rectify.py:124-129."""
    qv, qt, k, v = O.random_problem(4, t_v=64, t_t=9, d=16, dtype=np.float32)
    res = run_np(qv, qt, k, v, 8, 1.0, 0.0, 0, False, "sparse-rectified")
    _, full = O.full_attention_fp64(np.concatenate([qv, qt]), k, v)
    got = np.concatenate([res.output.o_video, res.output.o_text]).astype(np.float64)
    assert np.abs(got - full).max() <= 1e-5


def test_errors_map_to_reference_classes():
    qv, qt, k, v = O.random_problem(0, t_v=8, t_t=0, d=8)
    with pytest.raises(rsa.ConfigError):
        run_np(qv, qt, k, v, 4, 0.2, 0.3, 1, True, "bogus")


# ---------------------------------------------------------------- tcgen05 kernel

@pytest.mark.parametrize("d,block", [(64, 64), (64, 128), (128, 64), (128, 128)])
@pytest.mark.parametrize("t_t", [0, 1, 129, 200])
def test_tcgen05_kernel_matches_oracle_and_simt(d, block, t_t):
    """The tensor-core K3 against the fp32 oracle pipeline and the CUDA-core
    K3 on bf16-valued inputs: ragged text tile and ragged last kv block
    (t_t = 200), odd query-block count for B = 64, all retained lists."""
    heads = 2
    t_v = block * (23 if block == 64 else 12)
    rng = np.random.default_rng(d + block + t_t)
    per_head = []
    for h in range(heads):
        qv, qt, k, v = O.gen_synthetic(100 + h, t_v, max(t_t, 1), d, block, (1, 1, t_v), 1.0, 2.0, 0.3)
        qt, k, v = qt[:t_t], k[:t_v + t_t], v[:t_v + t_t]
        per_head.append(tuple(O.round_to_bf16(x) for x in (qv, qt, k, v)))
    q = torch.stack([torch.cat([to_bf16_tensor(a), to_bf16_tensor(b)]) for a, b, _, _ in per_head])
    k = torch.stack([to_bf16_tensor(x[2]) for x in per_head])
    v = torch.stack([to_bf16_tensor(x[3]) for x in per_head])
    outs = {}
    for kern in ("tcgen05", "simt"):
        lse = torch.empty(heads, t_v + t_t, dtype=torch.float32, device="cuda")
        outs[kern] = (rsa.rectified_sparse_attention(q, k, v, num_text_tokens=t_t, block=block,
                                                     top_k_fraction=0.2, weight_threshold=0.3,
                                                     adjacency_radius=1, force_text_blocks=True,
                                                     kernel=kern, lse=lse, check_status=True), lse)
    diff = (outs["tcgen05"][0].float() - outs["simt"][0].float()).abs().max().item()
    assert diff <= 1e-2, diff
    lse_diff = (outs["tcgen05"][1] - outs["simt"][1]).abs().max().item()
    assert lse_diff <= 1e-2, lse_diff
    for h, (qv, qt, kk, vv) in enumerate(per_head):
        ref = O.pipeline(qv, qt, kk, vv, block, 0.2, 0.3, 1, True, "sparse-rectified")
        assert_bf16_close(outs["tcgen05"][0][h], np.concatenate([ref["o_video"], ref["o_text"]]), f"head {h}")
        np.testing.assert_allclose(outs["tcgen05"][1][h, :t_v].cpu().numpy(), ref["lse"], atol=2e-2, rtol=0)


def test_tcgen05_unrectified_block_sparse_seam():
    """kernel-only seam (kernel.py:65-117) on the tensor-core kernel vs the fp64
    masked oracle, bf16-valued inputs."""
    rng = np.random.default_rng(11)
    block, d, t_v, t_t = 128, 128, 128 * 10, 77
    qv, qt, k, v = (O.round_to_bf16(x) for x in O.random_problem(5, t_v=t_v, t_t=t_t, d=d, dtype=np.float32))
    n, m, last = O.block_geometry(t_v, t_t, block)
    mask = rng.random((n, m)) < 0.35
    mask[np.arange(n), np.arange(n)] = True
    grid = partition(AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=d, block=block))
    out, _ = rsa.block_sparse_attention(to_bf16_tensor(qv), to_bf16_tensor(k), to_bf16_tensor(v),
                                        mask, grid, kernel="tcgen05")
    _, expected = O.masked_attention_fp64(qv, k, v, mask, O.kv_lengths(n, m, block, last), block)
    assert_bf16_close(out, expected, "seam")


@pytest.mark.parametrize("block,d,n_q", [(64, 64, 150), (128, 128, 140)])
def test_tcgen05_split_k_text_chunks(block, d, n_q):
    """M > 128 kv blocks: every 128-row text tile of the tensor-core kernel is
    split into kv-block chunks whose partial (O, max, sum) text_combine_kernel
    merges.  Against the CUDA-core kernel and the fp32 oracle."""
    t_v, t_t = block * n_q, 200
    qv, qt, k, v = O.gen_synthetic(7, t_v, t_t, d, block, (1, 1, t_v), 1.0, 2.0, 0.3)
    qv, qt, k, v = (O.round_to_bf16(x) for x in (qv, qt, k, v))
    q = torch.cat([to_bf16_tensor(qv), to_bf16_tensor(qt)])[None]
    kk, vv = to_bf16_tensor(k)[None], to_bf16_tensor(v)[None]
    outs = {}
    for kern in ("tcgen05", "simt"):
        lse = torch.empty(1, t_v + t_t, dtype=torch.float32, device="cuda")
        outs[kern] = (rsa.rectified_sparse_attention(q, kk, vv, num_text_tokens=t_t, block=block,
                                                     top_k_fraction=0.1, kernel=kern, lse=lse,
                                                     check_status=True)[0], lse[0])
    text = slice(t_v, t_v + t_t)
    diff = (outs["tcgen05"][0][text].float() - outs["simt"][0][text].float()).abs().max().item()
    assert diff <= 1e-2, diff
    lse_diff = (outs["tcgen05"][1][text] - outs["simt"][1][text]).abs().max().item()
    assert lse_diff <= 1e-2, lse_diff
    ref = O.pipeline(qv, qt, k, v, block, 0.1, 0.0, 0, False, "sparse-rectified")
    assert_bf16_close(outs["tcgen05"][0], np.concatenate([ref["o_video"], ref["o_text"]]), "split-K")


def test_forward_from_host_tensors_matches_device():
    """The end-to-end call on host tensors (rsa_forward_host: H2D, K1-K3, D2H
    pipelined over head chunks) returns exactly the device call's output."""
    heads, t_v, t_t, d, block = 3, 64 * 30, 100, 64, 64
    g = torch.Generator().manual_seed(3)
    q, k, v = (torch.randn(1, heads, t_v + t_t, d, generator=g).to(torch.bfloat16) for _ in range(3))
    want = rsa.rectified_sparse_attention(q.cuda(), k.cuda(), v.cuda(), num_text_tokens=t_t, block=block,
                                          top_k_fraction=0.2).cpu()
    for pinned, chunk in ((True, 1), (True, 2), (False, 3)):
        args = [x.pin_memory() if pinned else x for x in (q, k, v)]
        got = rsa.rectified_sparse_attention(*args, num_text_tokens=t_t, block=block, top_k_fraction=0.2,
                                             heads_per_chunk=chunk)
        assert not got.is_cuda
        assert torch.equal(got, want), (pinned, chunk)


def test_tcgen05_persistent_many_tiles_per_cta():
    """More 128-row tiles than SMs (each persistent CTA walks several tiles of
    several heads, text chunks and video tiles mixed): tensor-core output and
    LSE against the CUDA-core kernel, and bitwise repeatable."""
    heads, block, d, n_q, t_t = 5, 64, 64, 150, 77
    t_v = block * n_q
    g = torch.Generator().manual_seed(12)
    q, k, v = (torch.randn(heads, t_v + t_t, d, generator=g).to(torch.bfloat16).cuda() for _ in range(3))
    outs = {}
    for kern in ("tcgen05", "simt", "tcgen05"):
        lse = torch.empty(heads, t_v + t_t, dtype=torch.float32, device="cuda")
        o = rsa.rectified_sparse_attention(q, k, v, num_text_tokens=t_t, block=block, top_k_fraction=0.15,
                                           kernel=kern, lse=lse, check_status=True)
        if kern in outs:
            assert torch.equal(o, outs[kern][0]) and torch.equal(lse, outs[kern][1])
        outs[kern] = (o, lse)
    diff = (outs["tcgen05"][0].float() - outs["simt"][0].float()).abs().max().item()
    assert diff <= 1e-2, diff
    assert (outs["tcgen05"][1] - outs["simt"][1]).abs().max().item() <= 1e-2


# ---------------------------------------------------------------- K2 row kernels

@pytest.mark.parametrize("block,n_q,t_t,f,p,radius,force", [
    (16, 1400, 20, 0.1, 0.0, 0, False),    # 1,422 score columns: 12 per thread
    (24, 1700, 30, 0.3, 0.0, 2, True),     # 1,732 columns: 16 per thread; B=24 leaves pooling deficits
    (24, 1700, 30, 0.1, 0.4, 1, False),    # p > 0: the general (sorted-cumsum) row kernel
])
def test_select_rows_wide_rows_vs_oracle(block, n_q, t_t, f, p, radius, force):
    """K2 at row widths the HunyuanVideo shape does not reach (and a block size
    with non-zero pooling deficits, so the GAPR error term is live): masks,
    importance and the gain>error gate bit-exact, a_pool and R to 1e-12."""
    d = 32
    qv, qt, k, v = O.random_problem(7, t_v=block * n_q, t_t=t_t, d=d, dtype=np.float32)
    res = run_np(qv, qt, k, v, block, f, p, radius, force, "sparse-rectified")
    pooled = O.pool(qv, k, v, t_t, block)
    imp = O.implicit_attention(pooled, d, block, t_t)
    sel = O.select_mask(imp["a_pool"], f, p, radius, force, pooled["n_q"])
    comp = O.gain(O.pooled_scores(pooled, d), block, pooled["lens"]) > \
        O.pooling_error(qv, k, pooled, block, d)
    np.testing.assert_array_equal(res.sparse_mask.mask, sel["mask"])
    np.testing.assert_array_equal(res.sparse_mask.importance, sel["importance"])
    np.testing.assert_array_equal(res.comp_mask.mask, comp)
    np.testing.assert_allclose(res.implicit.a_pool, imp["a_pool"], atol=1e-12, rtol=0)
    np.testing.assert_allclose(res.factors.r, O.rect_factors(imp["a_pool"], sel["mask"]), atol=1e-12, rtol=0)


@pytest.mark.parametrize("p", [0.0, 0.5])
def test_select_rows_max_kv_blocks(p):
    """The C ABI's upper bound, M = 8192 kv blocks (T_v = 65,536 at B = 8): the
    general row kernel's shared memory fits with the cumulative-weight sort
    (p > 0) too; a sample of rows bit-exact against the oracle (rows are
    independent in a3-a7, so the oracle runs on the sampled q_pool rows only)."""
    block, d, n_q = 8, 8, 8192
    qv, qt, k, v = O.random_problem(9, t_v=block * n_q, t_t=0, d=d, dtype=np.float32)
    res = run_np(qv, qt, k, v, block, 0.1, p, 0, False, "sparse-rectified")
    rows = np.linspace(0, n_q - 1, 48).astype(int)
    pooled = O.pool(qv, k, v, 0, block)
    # T_t = 0: a_pool = the mixed softmax itself (ipar.py:59-60 identity bypass)
    a_pool = O.softmax_rows((pooled["q_pool"][rows] @ pooled["k_mix"].T) / np.sqrt(d))
    sel = O.select_mask(a_pool, 0.1, p, 0, False, n_q)
    # (select_mask's adjacency band indexes the sampled rows 0..47: compare the
    # importance set and add the diagonal (radius 0) at the true row indices)
    np.testing.assert_array_equal(res.sparse_mask.importance[rows], sel["importance"])
    want = sel["importance"].copy()
    want[np.arange(rows.size), rows] = True
    np.testing.assert_array_equal(res.sparse_mask.mask[rows], want)
    np.testing.assert_allclose(res.implicit.a_pool[rows], a_pool, atol=1e-12, rtol=0)
    with pytest.raises(rsa.NativeError):
        # one block more than the bound
        run_np(np.concatenate([qv, qv[:8]]), qt, np.concatenate([k, k[:8]]), np.concatenate([v, v[:8]]),
               block, 0.1, p, 0, False, "sparse-rectified")


@pytest.mark.parametrize("d,block", [(64, 64), (128, 128)])
@pytest.mark.parametrize("scale_range", [0, 24])
def test_bf16_pooling_bit_exact(scale_range, d, block):
    """K1's bf16 path (fp64 sums proven exact by the block's magnitude range,
    TwoSum otherwise) reproduces math.fsum means bit for bit; scale_range > 0
    spreads the rows over 2^+-scale_range so the range test and its fallback run."""
    rng = np.random.default_rng(17)
    t_v, t_t = block * 24, 100
    qv, qt, k, v = (O.round_to_bf16(x) for x in O.random_problem(3, t_v=t_v, t_t=t_t, d=d, dtype=np.float32))
    if scale_range:
        sc = lambda x: O.round_to_bf16(x * np.exp2(rng.integers(-scale_range, scale_range + 1, size=(x.shape[0], 1))))
        qv, qt, k, v = sc(qv), sc(qt), sc(k), sc(v)
    res = rsa.rectified_attention_pipeline(bf16_problem(qv, qt, k, v, block), SparsityConfig(0.2, 0.0, 0, False))
    ref = O.pool(qv, k, v, t_t, block)
    np.testing.assert_array_equal(res.pooled.q_pool.cpu().numpy(), ref["q_pool"])
    np.testing.assert_array_equal(res.pooled.v_pool.cpu().numpy(), ref["v_pool"])
    np.testing.assert_array_equal(res.pooled.k_mix_pool.cpu().numpy(), ref["k_mix"])


@pytest.mark.parametrize("d,block,t_t", [(64, 64, 100), (128, 128, 131)])
def test_bf16_pooling_bit_exact_hard_cases(d, block, t_t):
    """K1 against math.fsum on blocks built to break naive summation: exact
    zeros (the nonzero-minimum path), bf16 subnormals, 2^+-40 and 2^-120 magnitudes in
    one column with exact cancellations (the Shewchuk fallback must round
    correctly, where a (hi, lo) TwoSum merge need not), rows that are all zero,
    and a ragged text block (len 3 at d 128, B 128: non-power-of-two mean and
    deficit, compared bitwise through q_def / k_def via the GAPR error)."""
    rng = np.random.default_rng(23)
    t_v = block * 12
    qv, qt, k, v = (O.round_to_bf16(x) for x in O.random_problem(4, t_v=t_v, t_t=t_t, d=d, dtype=np.float32))
    big = np.float32(2.0 ** 40)
    for x in (qv, k, v):
        x[rng.random(x.shape) < 0.2] = 0.0                                  # exact zeros
        x[block:2 * block] = 0.0                                            # an all-zero block
        x[2 * block:2 * block + 5, :] *= np.float32(2.0 ** -120)            # subnormal bf16 values
        x[3 * block, :] = big                                               # big + ... - big:
        x[3 * block + 1, :] = -big                                          # cancels exactly
        x[3 * block + 2, :] = O.round_to_bf16(np.float32(3.0) * np.float32(2.0 ** -60))
        x[4 * block:4 * block + 3, :] = O.round_to_bf16(rng.standard_normal((3, d)).astype(np.float32) * big)
    qv, qt, k, v = (O.round_to_bf16(x) for x in (qv, qt, k, v))
    res = rsa.rectified_attention_pipeline(bf16_problem(qv, qt, k, v, block), SparsityConfig(0.2, 0.0, 0, False))
    ref = O.pool(qv, k, v, t_t, block)
    np.testing.assert_array_equal(res.pooled.q_pool.cpu().numpy(), ref["q_pool"])
    np.testing.assert_array_equal(res.pooled.v_pool.cpu().numpy(), ref["v_pool"])
    np.testing.assert_array_equal(res.pooled.k_mix_pool.cpu().numpy(), ref["k_mix"])
    np.testing.assert_array_equal(res.comp_mask.mask.cpu().numpy(),
                                  O.pipeline(qv, qt, k, v, block, 0.2, 0.0, 0, False)["comp"])


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
@pytest.mark.parametrize("where", ["q_video", "k", "v"])
def test_non_finite_inputs_raise_shape_error(dtype, where):
    """core.py:23-31 (check_matrix): inf / NaN in q/k/v is a ShapeError.  For
    CUDA tensors K1 flags it while pooling; the pipeline and the batched op
    (check_status=True) raise it from the device status."""
    qv, qt, k, v = O.random_problem(2, t_v=64 * 4, t_t=10, d=64, dtype=np.float32)
    arrs = {"q_video": qv, "q_text": qt, "k": k, "v": v}
    bad = arrs[where].copy()
    bad[5, 7] = np.nan if where != "v" else np.inf
    arrs[where] = bad
    t = {n: torch.from_numpy(a).to(dtype).cuda() for n, a in arrs.items()}
    prob = AttentionProblem(q_video=t["q_video"], q_text=t["q_text"], k=t["k"], v=t["v"], d=64, block=64)
    with pytest.raises(rsa.ShapeError):
        rsa.rectified_attention_pipeline(prob, SparsityConfig(0.5, 0.0, 0, False))
    if dtype == torch.bfloat16:
        q = torch.cat([t["q_video"], t["q_text"]])[None]
        with pytest.raises(rsa.ShapeError):
            rsa.rectified_sparse_attention(q, t["k"][None], t["v"][None], num_text_tokens=10, block=64,
                                           sparsity=0.5, check_status=True)


@pytest.mark.parametrize("heads", [1, 15])
def test_pair_pingpong_and_persistent_k3_agree(heads):
    """d = B = 128 runs the paired-tile K3 by default; kernel="tcgen05-pingpong"
    and "tcgen05-persistent" select the two-slot ping-pong and the one-tile
    persistent K3 (cross-checks, never chosen silently): all within the bf16
    bar of each other and of the oracle.  23 tiles per head (2 text + 21
    video): an odd tile count (the last pair has one tile), and at 15 heads
    (345 tiles) CTAs run two pairs that straddle heads and the text/video
    boundary."""
    qv, qt, k, v = (O.round_to_bf16(x) for x in O.gen_synthetic(5, 128 * 21, 200, 128, 128, (1, 42, 64), 1.0, 2.0, 0.3))
    q = torch.cat([to_bf16_tensor(qv), to_bf16_tensor(qt)])[None].expand(heads, -1, -1).contiguous()
    kk = to_bf16_tensor(k)[None].expand(heads, -1, -1).contiguous()
    vv = to_bf16_tensor(v)[None].expand(heads, -1, -1).contiguous()
    outs = {}
    for kern in ("tcgen05", "tcgen05-pingpong", "tcgen05-persistent"):
        o = rsa.rectified_sparse_attention(q, kk, vv, num_text_tokens=200, block=128, top_k_fraction=0.2,
                                           kernel=kern).float().cpu().numpy().astype(np.float64)
        assert all(np.array_equal(o[0], o[h]) for h in range(heads)), kern   # identical heads
        outs[kern] = o[0]
    assert np.abs(outs["tcgen05"] - outs["tcgen05-persistent"]).max() <= 2e-2
    assert np.abs(outs["tcgen05"] - outs["tcgen05-pingpong"]).max() <= 2e-2
    ref = O.pipeline(qv, qt, k, v, 128, 0.2, 0.0, 0, False, "sparse-rectified")
    want = np.concatenate([ref["o_video"], ref["o_text"]])
    for kern, got in outs.items():
        assert_bf16_close(got, want, kern)
