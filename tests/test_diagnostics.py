"""Validation diagnostics (reference masks.py:189-219, metrics.py:90-124):
the oracle restatement bit-exact against reference goldens (CPU), and the GPU
implementation (K1 + K2 + rsa_diagnostics, fp64) against them (GPU)."""

from pathlib import Path

import numpy as np
import pytest

from oracle import rsa_oracle as O

GOLDEN = Path(__file__).parent / "golden"
CASES = ((3, 96, 20, 16, 8), (5, 128, 0, 8, 16), (7, 64, 37, 32, 16))   # make_golden.DIAG_CASES


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN / "diagnostics.npz")


@pytest.mark.parametrize("case", CASES)
def test_oracle_diagnostics_match_reference(gold, case):
    seed, t_v, t_t, d, b = case
    qv, qt, k, v = O.random_problem(seed, t_v=t_v, t_t=t_t, d=d)
    p = O.pool(qv, k, v, t_t, b)
    sp = O.pooled_scores(p, d)
    eg, ee = O.exact_gain_error(qv, k, sp, b, p["lens"])
    ss, ssp, frac = O.denominator_report(qv, k, sp, b, p["lens"])
    g, e = O.gain(sp, b, p["lens"]), O.pooling_error(qv, k, p, b, d)
    tag = f"s{seed}"
    for name, got in (("gain", g), ("error", e), ("exact_gain", eg), ("exact_error", ee), ("s_sum", ss),
                      ("s_sum_pool", ssp)):
        assert np.array_equal(got, gold[f"{tag}_{name}"]), name
    assert frac == float(gold[f"{tag}_satisfied"])
    assert O.gapr_agreement(g, e, eg, ee) == float(gold[f"{tag}_agreement"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_diagnostics_match_reference(gold, case):
    import paper_2511_19835_b200 as rsa
    seed, t_v, t_t, d, b = case
    qv, qt, k, v = O.random_problem(seed, t_v=t_v, t_t=t_t, d=d)
    prob = rsa.AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=d, block=b)
    ge = rsa.gain_error(prob, with_exact=True)
    rep = rsa.denominator_equivalence_report(prob)
    tag = f"s{seed}"
    for name, got in (("gain", ge.gain), ("error", ge.error), ("exact_gain", ge.exact_gain),
                      ("exact_error", ge.exact_error), ("s_sum", rep.s_sum), ("s_sum_pool", rep.s_sum_pool)):
        want = gold[f"{tag}_{name}"]
        np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-13, err_msg=name)
    assert rep.satisfied_fraction == float(gold[f"{tag}_satisfied"])
    assert rsa.gapr_condition_agreement(prob) == float(gold[f"{tag}_agreement"])


@pytest.mark.gpu
def test_gpu_diagnostics_bf16_cfg1_scale():
    """bf16 inputs at the cfg1 shape (3,840 + 256 tokens, d = 64, B = 64) against
    the fp64 oracle on the same bf16-valued inputs."""
    import torch

    import paper_2511_19835_b200 as rsa
    qv, qt, k, v = O.gen_synthetic(42, 3840, 256, 64, 64, (1, 60, 64), 1.0, 2.0, 0.3)
    qv, qt, k, v = (O.round_to_bf16(x) for x in (qv, qt, k, v))
    bf = lambda x: torch.from_numpy(x).to(torch.bfloat16).cuda()  # noqa: E731
    prob = rsa.AttentionProblem(q_video=bf(qv), q_text=bf(qt), k=bf(k), v=bf(v), d=64, block=64)
    ge = rsa.gain_error(prob, with_exact=True)
    p = O.pool(qv, k, v, 256, 64)
    sp = O.pooled_scores(p, 64)
    eg, ee = O.exact_gain_error(qv, k, sp, 64, p["lens"])
    np.testing.assert_allclose(ge.exact_gain.cpu().numpy(), eg, rtol=1e-10)
    np.testing.assert_allclose(ge.exact_error.cpu().numpy(), ee, rtol=1e-9)
    ss, ssp, frac = O.denominator_report(qv, k, sp, 64, p["lens"])
    rep = rsa.denominator_equivalence_report(prob)
    np.testing.assert_allclose(rep.s_sum.cpu().numpy(), ss, rtol=1e-10)
    np.testing.assert_allclose(rep.s_sum_pool.cpu().numpy(), ssp, rtol=1e-10)
    assert abs(rep.satisfied_fraction - frac) <= 1.0 / 3840
