"""Experiments on the GPU path: the reference harness's problem sources,
``run_experiment`` and ``sweep_sparsity`` with its report artefacts
(harness.py:36-126 generator, harness.py:127-174 config/loading,
harness.py:223-331 reports and sweeps, harness.py:334-348 ``save_problem``).

Every variant runs through this package's kernels (``harness.run_variants``:
the pipeline on the GPU, scored against the dense fp64 reference computed on
the GPU), so the same experiment the reference runs on a toy problem runs at
production size.  The artefacts keep the reference's formats -- one
``report_<variant>.json`` per variant (schema 1), ``experiment.csv`` /
``sweep.csv`` with the reference's columns and ``repr`` number formatting, and
a ``timings.json`` sidecar -- so downstream tooling reads them unchanged.
The floating-point columns agree with the reference's to the kernels'
precision, not byte for byte (different summation order).  SVG plots are out
of scope.
"""

from __future__ import annotations

import csv
import io
import json
import math
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np

from .core import VARIANTS, AttentionProblem, SparsityConfig
from .errors import ConfigError, IoError
from .rsat import read_rsat, write_rsat

REPORT_SCHEMA_VERSION = 1
# PRNG contract (harness.py:1-9): PCG64 through SeedSequence(seed), one child
# stream per tensor, spawned in this order
STREAM_NAMES = ("q_video_base", "q_video_noise", "k_video_base", "k_video_noise",
                "q_text", "k_text", "v")
CSV_FIELDS = ("top_k_fraction", "variant", "normalized_l1", "cosine_similarity",
              "sparsity", "flops_full", "flops_sparse", "flops_overhead",
              "gapr_agreement", "checks_passed")


@dataclass(frozen=True)
class SyntheticSpec:
    """Generator knobs (harness.py:36-66): locality strength (alpha), text key
    norm boost (beta), intra-block noise (sigma), precision single/double."""

    seed: int
    t_v: int = 256
    t_t: int = 16
    d: int = 32
    block: int = 8
    grid_dims: tuple = (4, 8, 8)
    locality_strength: float = 1.0
    text_norm_boost: float = 1.0
    intra_block_noise: float = 0.3
    precision: str = "single"

    def __post_init__(self):
        if min(self.t_v, self.t_t, self.d, self.block) < 1:
            raise ConfigError("all sizes must be >= 1")
        t, h, w = self.grid_dims
        if t * h * w != self.t_v:
            raise ConfigError(f"grid_dims product {t * h * w} != t_v={self.t_v}")
        if self.t_v % self.block:
            raise ConfigError(f"t_v={self.t_v} not divisible by block={self.block}")
        if self.locality_strength < 0 or self.intra_block_noise < 0:
            raise ConfigError("locality_strength and intra_block_noise must be >= 0")
        if self.text_norm_boost < 1:
            raise ConfigError(f"text_norm_boost must be >= 1, got {self.text_norm_boost}")
        if self.precision not in ("single", "double"):
            raise ConfigError(f"precision must be single or double, got {self.precision!r}")


def _sincos(coords: np.ndarray, dim: int) -> np.ndarray:
    half = dim // 2
    freqs = np.exp(-math.log(10000.0) * (2 * np.arange(half + dim % 2) / max(dim, 1)))
    ang = coords[:, None] * freqs[None, :]
    out = np.zeros((coords.shape[0], dim), dtype=np.float64)
    out[:, 0::2] = np.sin(ang)
    out[:, 1::2] = np.cos(ang[:, :half])
    return out


def positional_embedding(grid_dims, d: int) -> np.ndarray:
    """3-D sinusoidal embedding of the row-major (t, h, w) token grid
    (harness.py:69-89): d - 2*(d//3) dims for t, d//3 each for h and w."""
    t, h, w = grid_dims
    d_hw = d // 3
    coords = np.indices((t, h, w)).reshape(3, -1).astype(np.float64)
    return np.concatenate([_sincos(coords[0], d - 2 * d_hw), _sincos(coords[1], d_hw),
                           _sincos(coords[2], d_hw)], axis=1)


def gen_synthetic(spec: SyntheticSpec) -> AttentionProblem:
    """The reference's deterministic synthetic problem (harness.py:92-126),
    same PRNG streams, so the tensors are bit-identical to the reference's."""
    streams = [np.random.Generator(np.random.PCG64(s))
               for s in np.random.SeedSequence(spec.seed).spawn(len(STREAM_NAMES))]
    draw = dict(zip(STREAM_NAMES, streams))
    n_blocks, d = spec.t_v // spec.block, spec.d
    pos = spec.locality_strength * positional_embedding(spec.grid_dims, d)

    def video(base_name, noise_name):
        base = draw[base_name].standard_normal((n_blocks, d))
        noise = draw[noise_name].standard_normal((spec.t_v, d))
        return np.repeat(base, spec.block, axis=0) + spec.intra_block_noise * noise + pos

    q_video = video("q_video_base", "q_video_noise")
    k_video = video("k_video_base", "k_video_noise")
    q_text = draw["q_text"].standard_normal((spec.t_t, d))
    k_text = spec.text_norm_boost * draw["k_text"].standard_normal((spec.t_t, d))
    v = draw["v"].standard_normal((spec.t_v + spec.t_t, d))
    dt = np.float32 if spec.precision == "single" else np.float64
    return AttentionProblem(q_video=q_video.astype(dt), q_text=q_text.astype(dt),
                            k=np.concatenate([k_video, k_text]).astype(dt), v=v.astype(dt),
                            d=d, block=spec.block, grid_dims=tuple(spec.grid_dims))


@dataclass(frozen=True)
class ExperimentConfig:
    """A problem source (synthetic spec xor RSAT problem paths), the sparsity
    knobs and a variant set (harness.py:127-146)."""

    synthetic: SyntheticSpec | None = None
    problem_paths: dict | None = None
    sparsity: SparsityConfig = field(default_factory=SparsityConfig)
    variants: tuple = ("full", "sparse-unrectified", "sparse-rectified")
    output_dir: str | None = None
    morton_reorder: bool = False
    compute_gapr_agreement: bool = True

    def __post_init__(self):
        if (self.synthetic is None) == (self.problem_paths is None):
            raise ConfigError("exactly one of synthetic spec or problem paths is required")
        if not self.variants:
            raise ConfigError("at least one variant is required")
        for variant in self.variants:
            if variant not in VARIANTS:
                raise ConfigError(f"unknown variant {variant!r}, expected one of {VARIANTS}")


def load_problem(config: ExperimentConfig, device=None) -> AttentionProblem:
    """Synthetic or RSAT-manifest problem (harness.py:149-174); RSAT tensors are
    read straight into device memory (``rsat.load_problem``)."""
    if config.synthetic is not None:
        problem = gen_synthetic(config.synthetic)
    else:
        from .rsat import load_problem as load_rsat
        problem = load_rsat(config.problem_paths, device)
    if config.morton_reorder:
        from .reorder import reorder_morton
        problem, _ = reorder_morton(problem)
    return problem


def save_problem(problem: AttentionProblem, out_dir) -> dict:
    """RSAT files plus a problem.json manifest (harness.py:334-348)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    manifest = {}
    for name in ("q_video", "q_text", "k", "v"):
        x = getattr(problem, name)
        if hasattr(x, "detach"):
            x = x.detach().cpu().numpy()
        path = out / f"{name}.rsat"
        write_rsat(path, x)
        manifest[name] = str(path)
    manifest.update(d=problem.d, block=problem.block,
                    grid_dims=list(problem.grid_dims) if problem.grid_dims else None)
    _atomic_write_text(out / "problem.json", json.dumps(manifest, indent=2, sort_keys=True) + "\n")
    return manifest


def _atomic_write_text(path: Path, text: str) -> None:
    tmp = path.with_name(path.name + ".tmp")
    try:
        tmp.write_text(text)
        tmp.replace(path)
    except OSError as exc:
        raise IoError(f"cannot write {path}: {exc}") from exc


def report_row(top_k_fraction: float, report) -> dict:
    """One CSV row in the reference's formatting (harness.py:229-241)."""
    return {"top_k_fraction": repr(float(top_k_fraction)), "variant": report.variant,
            "normalized_l1": repr(report.normalized_l1),
            "cosine_similarity": repr(report.cosine_similarity),
            "sparsity": repr(report.sparsity), "flops_full": report.flops_full,
            "flops_sparse": report.flops_sparse, "flops_overhead": report.flops_overhead,
            "gapr_agreement": "" if report.gapr_agreement is None else repr(report.gapr_agreement),
            "checks_passed": int(report.checks_passed)}


def rows_to_csv(rows) -> str:
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=CSV_FIELDS, lineterminator="\n")
    w.writeheader()
    w.writerows(rows)
    return buf.getvalue()


def report_json(config: ExperimentConfig, report) -> str:
    """Schema-1 report of one variant (harness.py:253-270); no timings, so
    repeated runs give the same file."""
    payload = {
        "schema_version": REPORT_SCHEMA_VERSION, "variant": report.variant,
        "problem": asdict(config.synthetic) if config.synthetic else config.problem_paths,
        "sparsity_config": asdict(config.sparsity),
        "metrics": {"normalized_l1": report.normalized_l1, "cosine_similarity": report.cosine_similarity,
                    "sparsity": report.sparsity, "flops_full": report.flops_full,
                    "flops_sparse": report.flops_sparse, "flops_overhead": report.flops_overhead,
                    "gapr_agreement": report.gapr_agreement},
        "checks_passed": report.checks_passed,
    }
    return json.dumps(payload, indent=2, sort_keys=True) + "\n"


def run_experiment(config: ExperimentConfig) -> dict:
    """All variants on the GPU; then (only after every variant finished) one
    JSON report per variant, experiment.csv and timings.json (harness.py:273-294)."""
    from .harness import run_variants
    problem = load_problem(config)
    reports = run_variants(problem, config.sparsity, config.variants,
                           compute_gapr=config.compute_gapr_agreement)
    if config.output_dir is not None:
        out = Path(config.output_dir)
        out.mkdir(parents=True, exist_ok=True)
        for v in config.variants:
            _atomic_write_text(out / f"report_{v}.json", report_json(config, reports[v]))
        _atomic_write_text(out / "experiment.csv",
                           rows_to_csv([report_row(config.sparsity.top_k_fraction, reports[v])
                                        for v in config.variants]))
        timings = {v: reports[v].wall_time_ms for v in config.variants}
        _atomic_write_text(out / "timings.json", json.dumps(timings, indent=2, sort_keys=True) + "\n")
    return reports


def sweep_sparsity(config: ExperimentConfig, top_k_fractions) -> str:
    """The variant set at each retention fraction, descending (so sparsity
    increases down the file); returns the CSV text and writes sweep.csv +
    timings.json when the config has an output directory (harness.py:305-331)."""
    from .harness import run_variants
    if not top_k_fractions:
        raise ConfigError("top_k_fractions must be non-empty")
    for f in top_k_fractions:
        if not 0.0 < f <= 1.0:
            raise ConfigError(f"top_k_fraction must be in (0, 1], got {f}")
    problem = load_problem(config)
    rows, timings = [], {}
    base = config.sparsity
    for f in sorted(set(top_k_fractions), reverse=True):
        sp = SparsityConfig(top_k_fraction=f, weight_threshold=base.weight_threshold,
                            adjacency_radius=base.adjacency_radius, force_text_blocks=base.force_text_blocks)
        reports = run_variants(problem, sp, config.variants, compute_gapr=config.compute_gapr_agreement)
        for v in config.variants:
            rows.append(report_row(f, reports[v]))
            timings[f"{f}/{v}"] = reports[v].wall_time_ms
    text = rows_to_csv(rows)
    if config.output_dir is not None:
        out = Path(config.output_dir)
        out.mkdir(parents=True, exist_ok=True)
        _atomic_write_text(out / "sweep.csv", text)
        _atomic_write_text(out / "timings.json", json.dumps(timings, indent=2, sort_keys=True) + "\n")
    return text


def read_problem_arrays(paths: dict) -> dict:
    """Host copies of a manifest's tensors (for tools that want numpy)."""
    return {name: read_rsat(paths[name]) for name in ("q_video", "q_text", "k", "v")}
