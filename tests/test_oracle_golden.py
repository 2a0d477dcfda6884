"""Pins the CPU oracle (oracle/rsa_oracle.py) to the reference: its own golden
fixtures (scripts/gen_fixtures.py) and reference pipeline outputs captured by
tests/golden/make_golden.py.  CPU only."""

import json
import math

import numpy as np
import pytest
from scipy.special import softmax

from conftest import N_TINY, tiny_case
from oracle import rsa_oracle as O

VARIANTS = O.VARIANTS


# --- reference fixtures (pkg/scripts/gen_fixtures.py section 1/2) ---------------

def test_block_pool_fixture(ref_fixtures):
    x = np.random.default_rng(42).standard_normal((8, 4))
    np.testing.assert_allclose(O.exact_means(x, [4, 4]), ref_fixtures["block_pool_expected"],
                               rtol=1e-14, atol=0)


def test_full_attention_fixture(ref_fixtures):
    rng = np.random.default_rng(42)
    q, k, v = (rng.standard_normal(s) for s in ((6, 8), (10, 8), (10, 8)))
    w, o = O.full_attention_fp64(q, k, v)
    np.testing.assert_allclose(w, ref_fixtures["full_attention_weights"], atol=1e-14, rtol=0)
    np.testing.assert_allclose(o, ref_fixtures["full_attention_output"], atol=1e-14, rtol=0)


def test_masked_oracle_fixture(ref_fixtures):
    rng = np.random.default_rng(42)
    q = rng.standard_normal((16, 8))
    k = rng.standard_normal((16, 8))
    mask = np.eye(4, dtype=bool)
    w, _ = O.masked_attention_fp64(q, k, k, mask, [4] * 4, 4)
    np.testing.assert_allclose(w, ref_fixtures["masked_oracle_weights"], atol=1e-14, rtol=0)


def test_mixed_pooled_fixture(ref_fixtures):
    rng = np.random.default_rng(42)
    q_pool = rng.standard_normal((4, 8))
    k_mix = rng.standard_normal((7, 8))
    got = O.softmax_rows((q_pool @ k_mix.T) / math.sqrt(8))
    np.testing.assert_allclose(got, ref_fixtures["mixed_pooled_expected"], atol=1e-14, rtol=0)


def test_attention_gain_fixture(ref_fixtures):
    scores = np.random.default_rng(42).standard_normal((4, 4))
    np.testing.assert_array_equal(O.gain(scores, 4, [4] * 4), ref_fixtures["attention_gain_expected"])


def test_ipar_fixture_and_scalar(ref_fixtures):
    rng = np.random.default_rng(42)
    q_video = rng.standard_normal((32, 8))
    k = rng.standard_normal((38, 8))
    v = rng.standard_normal((38, 8))
    pooled = O.pool(q_video, k, v, 6, 4)
    imp = O.implicit_attention(pooled, 8, 4, 6)
    np.testing.assert_allclose(imp["a_pool"], ref_fixtures["ipar_a_pool_expected"], atol=1e-12, rtol=0)
    # blocked truth cosine (scalars.json, ipar_blocked_truth_cosine)
    w = softmax(q_video @ k.T / math.sqrt(8), axis=1)
    lens = [4] * 8 + [4, 2]
    st = O.kv_starts(lens)
    truth = np.array([[w[i * 4:(i + 1) * 4, st[m]:st[m + 1]].sum() / 4 for m in range(10)]
                      for i in range(8)])
    a = imp["a_pool"]
    cos = float(a.ravel() @ truth.ravel() / (np.linalg.norm(a) * np.linalg.norm(truth)))
    scalars = json.loads(bytes(ref_fixtures["scalars_json"]).decode())
    assert cos == pytest.approx(scalars["ipar_blocked_truth_cosine"], abs=1e-9)


def test_metric_scalars(ref_fixtures):
    rng = np.random.default_rng(42)
    a = rng.standard_normal((5, 4))
    b = rng.standard_normal((5, 4))
    scalars = json.loads(bytes(ref_fixtures["scalars_json"]).decode())
    assert O.normalized_l1(a, b) == pytest.approx(scalars["normalized_l1"], abs=1e-15)
    assert O.cosine(a, b) == pytest.approx(scalars["cosine_similarity"], abs=1e-15)


def test_generator_fixture(ref_fixtures):
    qv, qt, k, v = O.gen_synthetic(42, 256, 16, 32, 8, (4, 8, 8), 1.0, 2.0, 0.3)
    for name, arr in (("q_video", qv), ("q_text", qt), ("k", k), ("v", v)):
        np.testing.assert_array_equal(arr, ref_fixtures[f"synthetic_{name}"])


def test_demo_sweep_row(ref_fixtures):
    """First sparse rows of the byte-exact demo sweep (pkg/tests/fixtures/demo_sweep.csv)."""
    csv = bytes(ref_fixtures["demo_sweep_csv"]).decode().splitlines()
    header = csv[0].split(",")
    rows = [dict(zip(header, line.split(","))) for line in csv[1:]]
    qv, qt, k, v = O.gen_synthetic(42, 64, 8, 16, 8, (1, 8, 8), 1.0, 2.0, 0.3)
    _, ref = O.full_attention_fp64(np.concatenate([qv, qt]), k, v)
    for row in rows:
        if row["variant"] == "full":
            continue
        res = O.pipeline(qv, qt, k, v, 8, float(row["top_k_fraction"]), 0.3, 1, True, row["variant"])
        out = np.concatenate([res["o_video"], res["o_text"]])
        assert repr(O.normalized_l1(out, ref)) == row["normalized_l1"]
        assert repr(O.cosine(out, ref)) == row["cosine_similarity"]
        sp, ff, fs = O.sparsity_and_flops(res["mask"], res["lens"], 8, 16)
        assert (repr(sp), str(ff), str(fs)) == (row["sparsity"], row["flops_full"], row["flops_sparse"])


# --- reference pipeline goldens (tests/golden/make_golden.py) -------------------

@pytest.mark.parametrize("i", range(N_TINY))
def test_tiny_pipeline_matches_reference(tiny_golden, i):
    (qv, qt, k, v), m = tiny_case(tiny_golden, i)
    for variant in VARIANTS:
        res = O.pipeline(qv, qt, k, v, m["block"], m["f"], m["p"], m["r"], m["force"], variant)
        tag = f"c{i}_{variant}"
        np.testing.assert_array_equal(res["o_video"], tiny_golden[f"{tag}_o_video"])
        np.testing.assert_array_equal(res["o_text"], tiny_golden[f"{tag}_o_text"])
        np.testing.assert_array_equal(res["lse"], tiny_golden[f"{tag}_lse"])
        if variant == "sparse-rectified":
            np.testing.assert_array_equal(res["mask"], tiny_golden[f"c{i}_mask"])
            np.testing.assert_array_equal(res["importance"], tiny_golden[f"c{i}_importance"])
            np.testing.assert_array_equal(res["comp"], tiny_golden[f"c{i}_comp"])
            np.testing.assert_array_equal(res["r"], tiny_golden[f"c{i}_r"])
            np.testing.assert_array_equal(res["a_pool"], tiny_golden[f"c{i}_a_pool"])
            np.testing.assert_array_equal(res["pooled"]["q_pool"], tiny_golden[f"c{i}_q_pool"])
            np.testing.assert_array_equal(res["pooled"]["v_pool"], tiny_golden[f"c{i}_v_pool"])
            np.testing.assert_array_equal(res["pooled"]["k_mix"], tiny_golden[f"c{i}_k_mix"])


def cfg1_inputs(seed):
    qv, qt, k, v = O.gen_synthetic(seed, 3840, 256, 64, 64, (1, 60, 64), 1.0, 2.0, 0.3)
    return tuple(O.round_to_bf16(x) for x in (qv, qt, k, v))


@pytest.mark.parametrize("seed", [42, 43])
def test_cfg1_pipeline_matches_reference(cfg1_golden, seed):
    qv, qt, k, v = cfg1_inputs(seed)
    chk = [float(np.abs(x).astype(np.float64).sum()) for x in (qv, qt, k, v)]
    np.testing.assert_array_equal(chk, cfg1_golden[f"s{seed}_input_checksum"])
    for f in (0.5, 0.25, 0.1, 0.05):
        for p in (0.0, 0.5):
            for variant in ("sparse-rectified", "sparse-unrectified"):
                res = O.pipeline(qv, qt, k, v, 64, f, p, 0, False, variant)
                tag = f"s{seed}_f{f}_p{p}_{variant}"
                np.testing.assert_array_equal(res["o_video"][::32], cfg1_golden[f"{tag}_o_rows"])
                np.testing.assert_array_equal(res["o_text"][::8], cfg1_golden[f"{tag}_ot_rows"])
            np.testing.assert_array_equal(np.packbits(res["mask"], axis=1),
                                          cfg1_golden[f"s{seed}_f{f}_p{p}_mask"])
            np.testing.assert_array_equal(res["r"], cfg1_golden[f"s{seed}_f{f}_p{p}_r"])
    np.testing.assert_array_equal(res["a_pool"], cfg1_golden[f"s{seed}_a_pool"])
    np.testing.assert_array_equal(np.packbits(res["comp"], axis=1), cfg1_golden[f"s{seed}_comp"])


# --- known-answer tests from the reference suite ----------------------------------

def test_greedy_rule_kat():
    """pkg/tests/test_masks.py:33-36."""
    sel = O.select_mask(np.array([[0.5, 0.3, 0.2]]), 1 / 3, 0.7, 0, False, 1)
    np.testing.assert_array_equal(sel["importance"], [[True, True, False]])


def test_uniform_tie_break_kat():
    """pkg/tests/test_masks.py:38-49: ties resolve to ascending block index."""
    sel = O.select_mask(np.full((8, 8), 1 / 8), 0.25, 0.0, 1, False, 8)
    for n in range(8):
        adj = {m for m in (n - 1, n, n + 1) if 0 <= m < 8}
        assert set(np.flatnonzero(sel["mask"][n])) == adj | {0, 1}


def test_reallocation_kat():
    """pkg/tests/test_ipar.py:74-78 through the full IPAR composition."""
    pooled = {"q_pool": np.zeros((1, 2)), "k_mix": np.zeros((2, 2)), "n_q": 1, "n_kv": 2}
    imp = O.implicit_attention(pooled, 2, 4, 1)
    # a_mix = [0.5 | 0.5]; D = 4*0.5 + 0.5 = 2.5 -> [0.8 | 0.2]
    np.testing.assert_allclose(imp["a_pool"], [[0.8, 0.2]])


def test_power_of_two_error_is_zero():
    """pkg/tests/test_masks.py:121-126."""
    qv, qt, k, v = O.random_problem(7, t_v=32, t_t=8, d=8)
    pooled = O.pool(qv, k, v, 8, 8)
    np.testing.assert_array_equal(O.pooling_error(qv, k, pooled, 8, 8), 0.0)


def test_ragged_gain_kat():
    """pkg/tests/test_masks.py:108-111."""
    np.testing.assert_array_equal(O.gain(np.ones((2, 3)), 4, [4, 4, 2]), [[16, 16, 8]] * 2)


def test_rect_factor_kat():
    """pkg/tests/test_rectify.py:27-31."""
    np.testing.assert_allclose(O.rect_factors(np.array([[0.5, 0.3, 0.2]]),
                                              np.array([[True, True, False]])), [0.8])


def test_oracle_against_live_reference_when_present():
    """Extra pin when the reference tree is mounted (build container only)."""
    import sys
    from pathlib import Path
    src = Path("/root/reference/pkg/src")
    if not src.exists():
        pytest.skip("reference tree not present")
    sys.path.insert(0, str(src))
    import rectattn as rt
    for seed in range(4):
        qv, qt, k, v = O.random_problem(100 + seed, t_v=48, t_t=5 + seed, d=16, dtype=np.float32)
        prob = rt.AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=16, block=8)
        for variant in VARIANTS:
            ref = rt.rectified_attention_pipeline(prob, rt.SparsityConfig(0.3, 0.4, 1, True), variant)
            got = O.pipeline(qv, qt, k, v, 8, 0.3, 0.4, 1, True, variant)
            np.testing.assert_array_equal(got["o_video"], ref.output.o_video)
            np.testing.assert_array_equal(got["mask"], ref.sparse_mask.mask)


@pytest.mark.parametrize("tag", ["hv", "wan"])
def test_oracle_matches_reference_at_headline_shapes(tag):
    """The oracle restatement reproduces the reference's own outputs on one
    full HunyuanVideo / Wan 2.1 head bit for bit (mask, sampled video rows of
    64 query blocks, all text rows, row log-denominators) -- the pin for the
    GPU headline parity tests (test_headline_parity.py)."""
    from threadpoolctl import threadpool_limits
    from conftest import load_golden
    g = load_golden("headline_outputs.npz")
    if tag == "hv":
        inputs = O.gen_synthetic(42, 118784, 256, 128, 128, (29, 64, 64), 1.0, 2.0, 0.3)
    else:
        rng = np.random.default_rng(42)
        qv, k, v = (rng.standard_normal((75520, 128)).astype(np.float32) for _ in range(3))
        inputs = (qv, np.zeros((0, 128), dtype=np.float32), k, v)
    qv, qt, k, v = (O.round_to_bf16(x) for x in inputs)
    qb = g[f"{tag}_query_blocks"]
    with threadpool_limits(1):
        ref = O.pipeline(qv, qt, k, v, 128, 0.1, 0.0, 0, False, "sparse-rectified", query_blocks=qb)
    np.testing.assert_array_equal(np.packbits(ref["mask"], axis=1), g[f"{tag}_mask"])
    np.testing.assert_array_equal(ref["o_video"][g[f"{tag}_rows"]], g[f"{tag}_o_video_rows"])
    np.testing.assert_array_equal(ref["o_text"], g[f"{tag}_o_text"])
    lse_rows = (qb[:, None] * 128 + np.arange(128)[None, :]).ravel()
    np.testing.assert_array_equal(ref["lse"][lse_rows], g[f"{tag}_lse_blocks"])
