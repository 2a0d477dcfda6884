"""The reference harness's experiment layer over the GPU path
(harness.py:36-348, cli.py:17-177): the synthetic generator is bit-identical
to the reference's fixtures; run/sweep artefacts keep the reference's formats
and reproduce its golden demo sweep (structural columns exactly, the
floating-point metrics to the kernels' precision)."""

import csv
import io
import json

import numpy as np
import pytest

from paper_2511_19835_b200.errors import ConfigError
from paper_2511_19835_b200.experiment import (CSV_FIELDS, ExperimentConfig, SyntheticSpec, gen_synthetic,
                                              report_row, rows_to_csv, save_problem)
from paper_2511_19835_b200.harness import AlignmentReport
from paper_2511_19835_b200.rsat import read_rsat
from paper_2511_19835_b200 import SparsityConfig


def demo_spec(**kw):
    base = dict(seed=42, t_v=64, t_t=8, d=16, block=8, grid_dims=(1, 8, 8),
                locality_strength=1.0, text_norm_boost=2.0, intra_block_noise=0.3)
    base.update(kw)
    return SyntheticSpec(**base)


def test_generator_matches_reference_fixture(ref_fixtures):
    spec = SyntheticSpec(seed=42, t_v=256, t_t=16, d=32, block=8, grid_dims=(4, 8, 8),
                         locality_strength=1.0, text_norm_boost=2.0, intra_block_noise=0.3)
    prob = gen_synthetic(spec)
    for name in ("q_video", "q_text", "k", "v"):
        np.testing.assert_array_equal(getattr(prob, name), ref_fixtures[f"synthetic_{name}"])


@pytest.mark.parametrize("kw", [dict(t_v=63), dict(grid_dims=(1, 8, 7)), dict(text_norm_boost=0.5),
                                dict(precision="half"), dict(intra_block_noise=-1.0)])
def test_spec_validation(kw):
    with pytest.raises(ConfigError):
        demo_spec(**kw)


def test_config_validation():
    with pytest.raises(ConfigError):
        ExperimentConfig()
    with pytest.raises(ConfigError):
        ExperimentConfig(synthetic=demo_spec(), variants=("nope",))
    with pytest.raises(ConfigError):
        ExperimentConfig(synthetic=demo_spec(), variants=())


def test_csv_format_matches_reference_golden_rows(ref_fixtures):
    """Formatting only: rebuild the golden file's rows from its own numbers."""
    golden = bytes(ref_fixtures["demo_sweep_csv"]).decode()
    rows = list(csv.DictReader(io.StringIO(golden)))
    rebuilt = []
    for r in rows:
        rep = AlignmentReport(variant=r["variant"], normalized_l1=float(r["normalized_l1"]),
                              cosine_similarity=float(r["cosine_similarity"]), sparsity=float(r["sparsity"]),
                              flops_full=int(r["flops_full"]), flops_sparse=int(r["flops_sparse"]),
                              flops_overhead=int(r["flops_overhead"]),
                              gapr_agreement=float(r["gapr_agreement"]) if r["gapr_agreement"] else None,
                              checks_passed=bool(int(r["checks_passed"])))
        rebuilt.append(report_row(float(r["top_k_fraction"]), rep))
    assert rows_to_csv(rebuilt) == golden
    assert tuple(rows[0].keys()) == CSV_FIELDS


def test_save_problem_roundtrip(tmp_path):
    prob = gen_synthetic(demo_spec())
    manifest = save_problem(prob, tmp_path)
    assert json.loads((tmp_path / "problem.json").read_text()) == manifest
    for name in ("q_video", "q_text", "k", "v"):
        np.testing.assert_array_equal(read_rsat(manifest[name]), getattr(prob, name))
    assert manifest["grid_dims"] == [1, 8, 8] and manifest["block"] == 8


# ---------------------------------------------------------------- GPU

def _parse(text):
    return list(csv.DictReader(io.StringIO(text)))


@pytest.mark.gpu
def test_gpu_demo_sweep_reproduces_reference_golden(ref_fixtures):
    """pkg/tests/test_harness.py:146-152 on the GPU path."""
    from paper_2511_19835_b200.experiment import sweep_sparsity
    config = ExperimentConfig(synthetic=demo_spec(), sparsity=SparsityConfig(0.5, 0.3, 1, True),
                              variants=("full", "sparse-unrectified", "sparse-rectified"))
    got = _parse(sweep_sparsity(config, [0.5, 0.2, 0.1]))
    want = _parse(bytes(ref_fixtures["demo_sweep_csv"]).decode())
    assert len(got) == len(want)
    for g, w in zip(got, want):
        for key in ("top_k_fraction", "variant", "sparsity", "flops_full", "flops_sparse", "flops_overhead",
                    "gapr_agreement", "checks_passed"):
            assert g[key] == w[key], key
        assert float(g["normalized_l1"]) == pytest.approx(float(w["normalized_l1"]), abs=1e-6)
        assert float(g["cosine_similarity"]) == pytest.approx(float(w["cosine_similarity"]), abs=1e-7)


@pytest.mark.gpu
def test_gpu_cli_gen_run_sweep_artifacts(tmp_path, capsys):
    from paper_2511_19835_b200.cli import main
    prob_dir, out = tmp_path / "prob", tmp_path / "out"
    assert main(["gen", "--tv", "64", "--tt", "8", "--d", "16", "--block", "8", "--grid", "1,8,8",
                 "--out", str(prob_dir)]) == 0
    assert main(["run", "--problem", str(prob_dir), "--topk", "0.5", "--out", str(out), "--device", "cuda"]) == 0
    for v in ("full", "sparse-unrectified", "sparse-rectified"):
        rep = json.loads((out / f"report_{v}.json").read_text())
        assert rep["schema_version"] == 1 and rep["variant"] == v and rep["checks_passed"] is True
    rows = _parse((out / "experiment.csv").read_text())
    assert [r["variant"] for r in rows] == ["full", "sparse-unrectified", "sparse-rectified"]
    assert float(rows[2]["normalized_l1"]) < float(rows[1]["normalized_l1"])   # rectification helps
    assert json.loads((out / "timings.json").read_text()).keys() == {"full", "sparse-unrectified",
                                                                      "sparse-rectified"}
    capsys.readouterr()
    assert main(["sweep", "--problem", str(prob_dir), "--topk-list", "0.5,0.1", "--out", str(out)]) == 0
    text = capsys.readouterr().out
    assert text == (out / "sweep.csv").read_text()
    sp = [float(r["sparsity"]) for r in _parse(text) if r["variant"] == "sparse-rectified"]
    assert sp == sorted(sp)
    assert main(["run", "--problem", str(prob_dir), "--device", "cpu"]) == 2
