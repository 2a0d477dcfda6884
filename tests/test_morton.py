"""Morton (Z-order) token reordering, reference core.py:263-325 and the
harness's morton_reorder option (harness.py:172-173).

CPU: the oracle restatement and the library's host permutation against the
reference goldens (tests/golden/morton_perms.npz from make_golden.py, and the
reference's own fixture morton_perm_2_4_4).  GPU: reorder_morton's device row
moves bit-exact against the oracle, and the fused permuted pipeline (gather in
K1, scatter in the K3 epilogue) against the oracle pipeline run on the
reordered problem."""

from pathlib import Path

import numpy as np
import pytest

from oracle import rsa_oracle as O

GOLDEN = Path(__file__).parent / "golden"


@pytest.fixture(scope="module")
def perms():
    z = np.load(GOLDEN / "morton_perms.npz")
    ref = np.load(GOLDEN / "reference_fixtures.npz")
    out = {tuple(int(x) for x in k.split("_")[1:]): z[k].astype(np.int64) for k in z.files}
    out[(2, 4, 4, "fixture")] = ref["morton_perm_2_4_4"].astype(np.int64)
    return out


def test_oracle_morton_matches_reference_goldens(perms):
    for key, want in perms.items():
        assert np.array_equal(O.morton_permutation(key[:3]), want), key
    assert np.array_equal(O.morton_permutation((1, 2, 2)), [0, 1, 2, 3])   # test_core.py:201-202


def test_oracle_reorder_roundtrip_bit_exact():
    qv, qt, k, v = O.random_problem(6, t_v=32, t_t=5, d=4)
    rq, rqt, rk, rv, perm = O.reorder_morton(qv, qt, k, v, (2, 4, 4))
    inv = O.inverse_permutation(perm)
    assert np.array_equal(rq[inv], qv) and np.array_equal(rk[:32][inv], k[:32])
    assert np.array_equal(rk[32:], k[32:]) and np.array_equal(rv[:32][inv], v[:32])


def test_library_morton_permutation_matches_goldens(perms):
    import paper_2511_19835_b200 as rsa
    for key, want in perms.items():
        got = rsa.morton_permutation(key[:3])
        assert got.dtype == np.int64 and np.array_equal(got, want), key
    # the HunyuanVideo grid against the oracle restatement
    assert np.array_equal(rsa.morton_permutation((29, 64, 64)), O.morton_permutation((29, 64, 64)))
    inv = rsa.inverse_permutation(want)
    assert np.array_equal(want[inv], np.arange(want.shape[0]))


def test_library_morton_errors():
    import paper_2511_19835_b200 as rsa
    qv, qt, k, v = O.random_problem(7, t_v=8, t_t=0, d=4)
    with pytest.raises(rsa.MissingGridError):
        rsa.reorder_morton(rsa.AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=4, block=4))
    with pytest.raises(rsa.ShapeError):
        rsa.morton_permutation((0, 4, 4))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_reorder_morton_on_gpu_bit_exact(dtype):
    import paper_2511_19835_b200 as rsa
    qv, qt, k, v = O.random_problem(8, t_v=3 * 4 * 6, t_t=7, d=16, dtype=dtype)
    prob = rsa.AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=16, block=8, grid_dims=(3, 4, 6))
    got, perm = rsa.reorder_morton(prob)
    rq, rqt, rk, rv, want_perm = O.reorder_morton(qv, qt, k, v, (3, 4, 6))
    assert np.array_equal(perm, want_perm)
    for a, b in ((got.q_video, rq), (got.q_text, rqt), (got.k, rk), (got.v, rv)):
        assert isinstance(a, np.ndarray) and a.dtype == dtype and np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("block,d,grid", [(64, 64, (2, 40, 48)), (128, 128, (3, 32, 40))])
def test_fused_morton_pipeline_matches_oracle(block, d, grid):
    """rectified_sparse_attention(morton=True): masks of the reordered problem
    bit-exact, outputs (original token order) within the bf16 tolerance of the
    oracle pipeline run on the reordered problem and permuted back."""
    import ctypes as C

    import torch

    import paper_2511_19835_b200 as rsa
    from paper_2511_19835_b200 import _native as nat
    from paper_2511_19835_b200.pipeline import workspace_for
    t_v, t_t = grid[0] * grid[1] * grid[2], 200
    qv, qt, k, v = O.gen_synthetic(11, t_v, t_t, d, block, grid, 1.0, 2.0, 0.3)
    qv, qt, k, v = (O.round_to_bf16(x) for x in (qv, qt, k, v))
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda()  # noqa: E731
    q = torch.cat([bf(qv), bf(qt)])[None]
    shape = nat.make_shape(1, t_v, t_t, d, block, "bfloat16")
    ws = workspace_for(shape, "cuda")
    out = rsa.rectified_sparse_attention(q, bf(k)[None], bf(v)[None], num_text_tokens=t_t, block=block,
                                         top_k_fraction=0.1, grid_dims=grid, morton=True, workspace=ws,
                                         check_status=True)[0]
    rq, rqt, rk, rv, perm = O.reorder_morton(qv, qt, k, v, grid)
    ref = O.pipeline(rq, rqt, rk, rv, block, 0.1, 0.0, 0, False, "sparse-rectified")
    L = nat.layout(shape)
    n, m = t_v // block, ref["mask"].shape[1]
    bits = ws[L["mask_bits"]:L["mask_bits"] + n * m].view(n, m).cpu().numpy()
    assert np.array_equal((bits & 1) != 0, ref["mask"])
    want = np.empty((t_v + t_t, d), np.float64)
    want[perm] = ref["o_video"]            # back to the original token order
    want[t_v:] = ref["o_text"]
    got = out.float().cpu().numpy().astype(np.float64)
    err, cos = np.abs(got - want).max(), O.cosine(got, want)
    assert err <= 2e-2 and cos >= 0.999, (err, cos)
