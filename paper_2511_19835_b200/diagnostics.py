"""Validation diagnostics on the GPU (reference masks.py:189-219 and
metrics.py:90-124): the exact softmax-form GAPR terms, the relaxed/exact
compensation-condition agreement and the softmax-denominator equivalence
report.  Quadratic in sequence length like the reference's, computed in fp64
(K1 + K2, then rsa_diagnostics: cuBLAS DGEMM for S = QKᵀ per chunk of query
blocks and our reduction kernels), so they run at production sizes.

The reference functions take ``pooled`` / ``grid`` from ``pool_problem``; here
they are recomputed on the device and the arguments are accepted for
signature compatibility only."""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as nat
from .core import (AttentionProblem, DenominatorReport, GainError, SparsityConfig, _is_torch,
                   partition)


def _diagnose(problem: AttentionProblem):
    from .pipeline import _as_tensor, _device, _ptr, _stream, workspace_for
    dev = _device()
    grid = partition(problem)
    t_v, t_t, d = problem.t_v, problem.t_t, problem.d
    q = torch.cat([_as_tensor(problem.q_video, dev), _as_tensor(problem.q_text, dev)]).contiguous()
    k = _as_tensor(problem.k, dev).contiguous()
    shape = nat.make_shape(1, t_v, t_t, d, problem.block, str(q.dtype).replace("torch.", ""))
    cfg = nat.make_config(1.0, 0.0, 0, False, "sparse-rectified")   # the gate does not depend on it
    nat.plan(shape, cfg)
    ws = workspace_for(shape, dev)
    lib, st = nat.lib(), _stream()
    v = _as_tensor(problem.v, dev).contiguous()
    nat.check(lib.rsa_pool(C.byref(shape), _ptr(q), _ptr(k), _ptr(v), _ptr(ws), st))
    nat.check(lib.rsa_select(C.byref(shape), C.byref(cfg), _ptr(ws), st))
    n, m = grid.n_q, grid.n_kv
    f64 = dict(dtype=torch.float64, device=dev)
    out = {name: torch.empty(n, m, **f64) for name in ("gain", "error", "exact_gain", "exact_error")}
    out["s_sum"] = torch.empty(t_v, **f64)
    out["s_sum_pool"] = torch.empty(t_v, **f64)
    scratch = torch.empty(lib.rsa_diagnostics_scratch_size(C.byref(shape)), dtype=torch.uint8, device=dev)
    nat.check(lib.rsa_diagnostics(C.byref(shape), _ptr(q), _ptr(k), _ptr(ws),
                                  *(_ptr(out[x]) for x in ("gain", "error", "exact_gain", "exact_error",
                                                           "s_sum", "s_sum_pool")),
                                  _ptr(scratch), st))
    nat.check(lib.rsa_check_device_status(_ptr(ws), st))
    host = not _is_torch(problem.q_video)
    return {k_: (v_.cpu().numpy() if host else v_) for k_, v_ in out.items()}


def _fraction(flags) -> float:
    return float(flags.double().mean()) if _is_torch(flags) else float(flags.mean())


def gain_error(problem: AttentionProblem, pooled=None, grid=None, scores_pool=None,
               with_exact: bool = False) -> GainError:
    """Relaxed gain/error, optionally with the exact softmax forms. masks.py:189-219."""
    r = _diagnose(problem)
    if not with_exact:
        return GainError(gain=r["gain"], error=r["error"])
    return GainError(gain=r["gain"], error=r["error"], exact_gain=r["exact_gain"], exact_error=r["exact_error"])


def gapr_condition_agreement(problem: AttentionProblem, pooled=None, grid=None) -> float:
    """Fraction of blocks where the relaxed compensation condition agrees with
    the exact softmax-form one. metrics.py:116-124."""
    r = _diagnose(problem)
    relaxed = r["gain"] > r["error"]
    exact = r["exact_gain"] > r["exact_error"]
    return _fraction(relaxed == exact)


def denominator_equivalence_report(problem: AttentionProblem, pooled=None, grid=None,
                                   tau: float = 0.05) -> DenominatorReport:
    """True vs pooled softmax denominators of every video query token.
    metrics.py:90-113."""
    r = _diagnose(problem)
    s, sp = r["s_sum"], r["s_sum_pool"]
    satisfied = abs(s - sp) < tau * abs(s)
    return DenominatorReport(s_sum=s, s_sum_pool=sp, satisfied_fraction=_fraction(satisfied), tau=tau)
