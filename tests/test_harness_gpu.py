"""The reference harness's core (harness.py:177-220 run_variants, metrics.py
AlignmentReport / normalized_l1 / cosine_similarity) on the GPU, against the
reference's own run_variants results (tests/golden/harness_variants.npz)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import rsa_oracle as O

GOLDEN = Path(__file__).parent / "golden"
CASES = ((21, 128, 20, 16, 16, 0.25), (22, 256, 0, 32, 32, 0.1))   # make_golden.HARNESS_CASES
VARIANTS = ("full", "sparse-unrectified", "sparse-rectified", "sparse-rectified-no-gapr", "compensate-all")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", CASES)
def test_run_variants_matches_reference(case):
    import paper_2511_19835_b200 as rsa
    gold = np.load(GOLDEN / "harness_variants.npz")
    seed, t_v, t_t, d, b, f = case
    qv, qt, k, v = O.random_problem(seed, t_v=t_v, t_t=t_t, d=d)
    prob = rsa.AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=d, block=b)
    reps = rsa.run_variants(prob, rsa.SparsityConfig(f, 0.0, 0, False), VARIANTS)
    for name in VARIANTS:
        r, want = reps[name], gold[f"s{seed}_{name}"]
        np.testing.assert_allclose([r.normalized_l1, r.cosine_similarity], want[:2], rtol=1e-10, atol=1e-13,
                                   err_msg=name)
        assert r.sparsity == want[2] and (r.flops_full, r.flops_sparse, r.flops_overhead) == tuple(want[3:6])
        assert r.gapr_agreement == want[6] and r.checks_passed == bool(want[7])


def test_dense_reference_matches_oracle_bf16():
    """fp64 dense reference of bf16-valued inputs at the cfg1 shape vs numpy fp64."""
    import torch

    import paper_2511_19835_b200 as rsa
    qv, qt, k, v = O.gen_synthetic(42, 3840, 256, 64, 64, (1, 60, 64), 1.0, 2.0, 0.3)
    qv, qt, k, v = (O.round_to_bf16(x) for x in (qv, qt, k, v))
    bf = lambda x: torch.from_numpy(x).to(torch.bfloat16).cuda()  # noqa: E731
    prob = rsa.AttentionProblem(q_video=bf(qv), q_text=bf(qt), k=bf(k), v=bf(v), d=64, block=64)
    got = rsa.full_attention_reference(prob).cpu().numpy()
    w = O.full_weights_fp64(np.concatenate([qv, qt]), k)
    want = w @ v.astype(np.float64)
    np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-12)
