"""The reference harness's core on the GPU: score every variant of the call
against the dense fp64 ground truth (harness.py:177-220 run_variants,
metrics.py:19-68 AlignmentReport / normalized_l1 / cosine_similarity).

The dense reference (``full_attention_oracle``, core.py:211-225) is computed on
the device in fp64 (``rsa_dense_reference``: cuBLAS DGEMMs around our softmax
kernel), so the reference's accuracy experiment -- e.g. the rectified vs the
plain block-sparse error at a given sparsity -- runs at production sizes.
Sweeps, CSV/JSON artefacts and plots stay out of scope."""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .core import AttentionProblem, SparsityConfig, _is_torch, check_result_invariants, partition, \
    sparsity_and_flops
from .errors import ConfigError, ShapeError, ZeroReferenceError, ZeroVectorError


@dataclass
class AlignmentReport:
    """One variant's alignment and cost summary (metrics.py:19-32)."""

    variant: str
    normalized_l1: float
    cosine_similarity: float
    sparsity: float
    flops_full: int
    flops_sparse: int
    flops_overhead: int
    wall_time_ms: dict = field(default_factory=dict)
    gapr_agreement: float | None = None
    checks_passed: bool = True


def _f64(x) -> torch.Tensor:
    from .pipeline import _as_tensor, _device
    return _as_tensor(x, _device()).to(torch.float64)


def normalized_l1(test, reference) -> float:
    """Sum of absolute differences normalised by the reference magnitude (metrics.py:46-55)."""
    a, b = _f64(test), _f64(reference)
    if a.shape != b.shape:
        raise ShapeError(f"shapes disagree: {tuple(a.shape)} vs {tuple(b.shape)}")
    denom = b.abs().sum()
    if float(denom) == 0.0:
        raise ZeroReferenceError("reference matrix is all zero")
    return float((a - b).abs().sum() / denom)


def cosine_similarity(test, reference) -> float:
    """Cosine of the flattened matrices (metrics.py:58-68)."""
    a, b = _f64(test).ravel(), _f64(reference).ravel()
    if a.shape != b.shape:
        raise ShapeError(f"shapes disagree: {tuple(a.shape)} vs {tuple(b.shape)}")
    na, nb = torch.linalg.norm(a), torch.linalg.norm(b)
    if float(na) == 0.0 or float(nb) == 0.0:
        raise ZeroVectorError("cosine similarity of a zero vector is undefined")
    return float(a @ b / (na * nb))


def full_attention_reference(problem: AttentionProblem) -> torch.Tensor:
    """Dense fp64 attention of [q_video; q_text] over all keys (core.py:211-225),
    [T, d] float64 on the GPU."""
    from .pipeline import _as_tensor, _device, _ptr, _stream
    dev = _device()
    q = torch.cat([_as_tensor(problem.q_video, dev), _as_tensor(problem.q_text, dev)]).contiguous()
    k = _as_tensor(problem.k, dev).contiguous()
    v = _as_tensor(problem.v, dev).contiguous()
    shape = nat.make_shape(1, problem.t_v, problem.t_t, problem.d, problem.block,
                           str(q.dtype).replace("torch.", ""))
    out = torch.empty(q.shape, dtype=torch.float64, device=dev)
    scratch = torch.empty(nat.lib().rsa_dense_reference_scratch_size(C.byref(shape)), dtype=torch.uint8,
                          device=dev)
    nat.check(nat.lib().rsa_dense_reference(C.byref(shape), _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                            _ptr(scratch), _stream()))
    return out


def run_variants(problem: AttentionProblem, sparsity: SparsityConfig, variants,
                 compute_gapr: bool = True) -> dict:
    """Run each variant against the dense fp64 reference (harness.py:177-220).
    The ``full`` variant *is* the reference run: its error is zero by
    definition.  Returns ``{variant: AlignmentReport}``."""
    from .core import VARIANTS
    from .diagnostics import gapr_condition_agreement
    from .pipeline import rectified_attention_pipeline
    for variant in variants:
        if variant not in VARIANTS:
            raise ConfigError(f"unknown variant {variant!r}, expected one of {VARIANTS}")
    grid = partition(problem)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reference = full_attention_reference(problem)
    torch.cuda.synchronize()
    reference_ms = (time.perf_counter() - t0) * 1e3
    gapr = gapr_condition_agreement(problem) if compute_gapr else None
    reports = {}
    for variant in variants:
        if variant == "full":
            flops_dense = 4 * problem.t_v * int(problem.k.shape[0]) * problem.d
            reports[variant] = AlignmentReport(
                variant=variant, normalized_l1=normalized_l1(reference, reference),
                cosine_similarity=cosine_similarity(reference, reference), sparsity=0.0,
                flops_full=flops_dense, flops_sparse=flops_dense, flops_overhead=0,
                wall_time_ms={"reference": reference_ms}, gapr_agreement=gapr, checks_passed=True)
            continue
        result = rectified_attention_pipeline(problem, sparsity, variant=variant, timing=True)
        o_video, o_text = result.output.o_video, result.output.o_text
        output = (torch.cat([o_video, o_text]) if _is_torch(o_video)
                  else np.concatenate([o_video, o_text], axis=0))
        s_ratio, flops_full, flops_sparse, flops_overhead = sparsity_and_flops(result.sparse_mask, result.grid,
                                                                               problem.d)
        reports[variant] = AlignmentReport(
            variant=variant, normalized_l1=normalized_l1(output, reference),
            cosine_similarity=cosine_similarity(output, reference), sparsity=s_ratio,
            flops_full=flops_full, flops_sparse=flops_sparse, flops_overhead=flops_overhead,
            wall_time_ms=dict(result.accounting.stage_wall_ms), gapr_agreement=gapr,
            checks_passed=check_result_invariants(result))
    del grid
    return reports
