"""Host-side containers mirroring the reference's public types.

Same names, fields and validation as pkg/src/rectattn (core.py, masks.py,
ipar.py, kernel.py, rectify.py) so a caller of the reference can switch
imports.  Arrays may be numpy (float32/float64, the reference's types) or torch
tensors (bfloat16/float32/float64, any device); results come back in the kind
the caller passed in.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import BlockSizeError, ConfigError, ShapeError

try:  # torch is plumbing (device memory, streams); numpy-only callers still work
    import torch
except ImportError:  # pragma: no cover
    torch = None

VARIANTS = ("full", "sparse-unrectified", "sparse-rectified",
            "sparse-rectified-no-gapr", "compensate-all")   # rectify.py:23-24

_NP_DTYPES = (np.float32, np.float64)


def _is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def dtype_name(x) -> str:
    if _is_torch(x):
        return str(x.dtype).replace("torch.", "")
    return np.dtype(x.dtype).name


def check_matrix(x, name: str = "matrix"):
    """2-D float matrix with finite entries (core.py:23-31).  Torch tensors may
    also be bfloat16 (the tensor-core path)."""
    if _is_torch(x):
        if x.dim() != 2:
            raise ShapeError(f"{name} must be a 2-D tensor, got {x.dim()}-D")
        if x.dtype not in (torch.bfloat16, torch.float32, torch.float64):
            raise ShapeError(f"{name} must be bfloat16, float32 or float64, got {x.dtype}")
        # CUDA tensors: K1 flags inf / NaN while pooling (no extra pass, no host
        # sync here); the pipeline raises the same ShapeError from the device status
        if not x.is_cuda and x.numel() and not bool(torch.isfinite(x).all()):
            raise ShapeError(f"{name} contains non-finite entries")
        return x
    if not isinstance(x, np.ndarray) or x.ndim != 2:
        raise ShapeError(f"{name} must be a 2-D numpy array, got {type(x).__name__}")
    if x.dtype not in _NP_DTYPES:
        raise ShapeError(f"{name} must be float32 or float64, got {x.dtype}")
    if x.size and not np.isfinite(x).all():
        raise ShapeError(f"{name} contains non-finite entries")
    return x


@dataclass(frozen=True, eq=False)
class AttentionProblem:
    """One single-head attention call with a video/text split (core.py:42-91).
    ``k``/``v`` hold video rows first, then text rows."""

    q_video: object
    q_text: object
    k: object
    v: object
    d: int
    block: int
    grid_dims: tuple | None = None
    # extension: accept T_v % block != 0, the final
    # video block holding the remaining T_v - (N-1)*block tokens; the reference
    # raises BlockSizeError (core.py:71-72), which stays the default
    ragged_video: bool = False

    def __post_init__(self):
        for name in ("q_video", "q_text", "k", "v"):
            check_matrix(getattr(self, name), name)
        for name in ("q_video", "q_text", "k", "v"):
            if getattr(self, name).shape[1] != self.d:
                raise ShapeError(f"{name} has width {getattr(self, name).shape[1]}, expected d={self.d}")
        if self.k.shape[0] != self.t_v + self.t_t or self.v.shape[0] != self.t_v + self.t_t:
            raise ShapeError("k/v row counts must equal T_v + T_t")
        if self.block <= 0:
            raise BlockSizeError(f"block size must be positive, got {self.block}")
        if self.t_v % self.block != 0 and not self.ragged_video:
            raise BlockSizeError(f"T_v={self.t_v} is not divisible by block size {self.block}")
        if self.t_v == 0:
            raise ShapeError("T_v must be >= 1 block")
        kinds = {(_is_torch(m), dtype_name(m)) for m in (self.q_video, self.q_text, self.k, self.v)}
        if len(kinds) != 1:
            raise ShapeError(f"q/k/v dtypes disagree: {sorted(str(t) for t in kinds)}")
        if self.grid_dims is not None:
            t, h, w = self.grid_dims
            if t * h * w != self.t_v:
                raise ShapeError(f"grid_dims product {t * h * w} != T_v={self.t_v}")

    @property
    def t_v(self) -> int:
        return int(self.q_video.shape[0])

    @property
    def t_t(self) -> int:
        return int(self.q_text.shape[0])

    @property
    def dtype(self):
        return self.q_video.dtype


@dataclass(frozen=True)
class BlockGrid:
    """N query blocks, M key/value blocks (core.py:94-123)."""

    n_q: int
    n_kv: int
    block: int
    text_block_start: int
    last_text_block_len: int
    last_video_block_len: int | None = None   # None: block (ragged_video extension)

    @property
    def ragged(self) -> bool:
        return self.last_video_block_len not in (None, self.block)

    @property
    def t_video(self) -> int:
        return sum(self.q_block_lengths())

    def q_block_lengths(self) -> list[int]:
        last = self.block if self.last_video_block_len is None else self.last_video_block_len
        return [self.block] * (self.n_q - 1) + [last]

    def kv_block_lengths(self) -> list[int]:
        lens = self.q_block_lengths()
        n_text = self.n_kv - self.n_q
        if n_text:
            lens += [self.block] * (n_text - 1) + [self.last_text_block_len]
        return lens

    def kv_block_slices(self) -> list[slice]:
        out, start = [], 0
        for length in self.kv_block_lengths():
            out.append(slice(start, start + length))
            start += length
        return out

    @property
    def t_text(self) -> int:
        n_text = self.n_kv - self.n_q
        return 0 if n_text == 0 else (n_text - 1) * self.block + self.last_text_block_len


def partition(problem: AttentionProblem) -> BlockGrid:
    """N = T_v / B, M = N + ceil(T_t / B) (core.py:140-151)."""
    b = problem.block
    if b <= 0:
        raise BlockSizeError(f"block size must be positive, got {b}")
    if problem.t_v % b != 0 and not getattr(problem, "ragged_video", False):
        raise BlockSizeError(f"T_v={problem.t_v} is not divisible by block size {b}")
    n_q = -(-problem.t_v // b)
    n_text = -(-problem.t_t // b)
    last = problem.t_t - (n_text - 1) * b if n_text else 0
    return BlockGrid(n_q=n_q, n_kv=n_q + n_text, block=b, text_block_start=n_q,
                     last_text_block_len=last,
                     last_video_block_len=problem.t_v - (n_q - 1) * b if problem.t_v % b else None)


@dataclass(frozen=True)
class SparsityConfig:
    """Knobs of the sparse mask (masks.py:21-41)."""

    top_k_fraction: float = 0.2
    weight_threshold: float = 0.3
    adjacency_radius: int = 1
    force_text_blocks: bool = True

    def __post_init__(self):
        if not 0.0 < self.top_k_fraction <= 1.0:
            raise ConfigError(f"top_k_fraction must be in (0, 1], got {self.top_k_fraction}")
        if not 0.0 <= self.weight_threshold <= 1.0:
            raise ConfigError(f"weight_threshold must be in [0, 1], got {self.weight_threshold}")
        if self.adjacency_radius < 0:
            raise ConfigError(f"adjacency_radius must be >= 0, got {self.adjacency_radius}")

    @classmethod
    def from_sparsity(cls, sparsity: float) -> "SparsityConfig":
        """Convenience: a target sparsity s maps to top-k fraction 1 - s with no
        threshold, band or forced text.  The always-kept diagonal
        (masks.py:111) makes the realized sparsity slightly lower."""
        return cls(top_k_fraction=1.0 - float(sparsity), weight_threshold=0.0,
                   adjacency_radius=0, force_text_blocks=False)


@dataclass(frozen=True, eq=False)
class PooledSet:
    """core.py:126-137."""

    q_pool: object
    k_v_pool: object
    v_pool: object
    k_mix_pool: object


class ImplicitAttention:
    """Block-level implicit full attention (ipar.py:18-33).  ``a_pool`` is the
    kernel output; the pre-reallocation intermediates are recomputed on demand
    from the fp64 pooled scores (diagnostics only, never on the hot path)."""

    def __init__(self, a_pool, scores_mix, n_q: int, block: int, t_t: int, to_host):
        self.a_pool = a_pool
        self._scores_mix = scores_mix
        self._n_q, self._block, self._t_t = n_q, block, t_t
        self._to_host = to_host
        self._cache = None

    def _intermediates(self):
        if self._cache is None:
            s = self._scores_mix
            a_mix = torch.softmax(s, dim=1) if _is_torch(s) else _np_softmax(s)
            n = self._n_q
            a_v, a_t = a_mix[:, :n], a_mix[:, n:]
            if a_t.shape[1] and self._block != 1:
                den = self._block * a_v.sum(1) + a_t.sum(1)
                a_v, a_t = self._block * a_v / den[:, None], a_t / den[:, None]
            self._cache = tuple(self._to_host(x) for x in (a_mix, a_v, a_t))
        return self._cache

    @property
    def a_mix_pool(self):
        return self._intermediates()[0]

    @property
    def a_v_reallocated(self):
        return self.a_pool[:, :self._n_q]

    @property
    def a_t_reallocated(self):
        return self._intermediates()[2]

    @property
    def a_t_block(self):
        return self.a_pool[:, self._n_q:]


def _np_softmax(s):
    e = np.exp(s - s.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


@dataclass(frozen=True, eq=False)
class SparseMask:
    """masks.py:44-55."""

    mask: object
    importance: object
    adjacency: object
    retained_count: object

    @property
    def retained_total(self) -> int:
        return int(self.mask.sum())


@dataclass(frozen=True, eq=False)
class GainError:
    """Relaxed-form gain and pooling error per block, with the optional exact
    softmax-form values kept for validation (masks.py:58-66)."""

    gain: object
    error: object
    exact_gain: object | None = None
    exact_error: object | None = None


@dataclass(frozen=True, eq=False)
class DenominatorReport:
    """Per-video-token softmax denominators, true vs pooled, and the fraction
    within a relative threshold of each other (metrics.py:35-43)."""

    s_sum: object
    s_sum_pool: object
    satisfied_fraction: float
    tau: float


@dataclass(frozen=True, eq=False)
class CompensationMask:
    """masks.py:69-73: consumed as ``~sparse.mask & mask``."""

    mask: object


@dataclass(frozen=True, eq=False)
class RectificationFactors:
    """rectify.py:27-31."""

    r: object


@dataclass(frozen=True, eq=False)
class AttentionOutput:
    """kernel.py:21-29."""

    o_video: object
    o_text: object
    row_log_denominators: object


@dataclass
class PipelineAccounting:
    """rectify.py:34-40."""

    stage_ops: dict = field(default_factory=dict)
    kernel_inner_product_ops: int = 0
    stage_wall_ms: dict = field(default_factory=dict)


@dataclass(frozen=True, eq=False)
class PipelineResult:
    """rectify.py:43-53."""

    output: AttentionOutput
    factors: RectificationFactors
    implicit: ImplicitAttention
    sparse_mask: SparseMask
    comp_mask: CompensationMask
    accounting: PipelineAccounting
    grid: BlockGrid
    pooled: PooledSet
    variant: str


def stage_op_counts(grid: BlockGrid, d: int) -> dict:
    """Multiply-add counts of the pooled path per stage (rectify.py:179-193)."""
    n, m, b = grid.n_q, grid.n_kv, grid.block
    t_v = grid.t_video
    t_t = grid.t_text
    t = t_v + t_t
    return {
        "pooling": 2 * d * (2 * t_v + t + t_t),
        "pooled_softmax": 2 * n * (n + t_t) * d + 4 * n * (n + t_t) + 2 * n * (n + t_t) + n * t_t,
        "gain_error": 2 * n * m * d + 2 * n * m + 2 * (n + m) * d + 4 * n * m * d + 3 * n * m + n * m,
        "compensation": n * m + 2 * n * m * d + 2 * t_v * d + n * m,
    }


def check_result_invariants(result: PipelineResult, tol: float = 1e-6) -> bool:
    """rectify.py:92-104 (host-side, on the returned arrays)."""
    to_np = lambda x: x.detach().cpu().numpy() if _is_torch(x) else np.asarray(x)  # noqa: E731
    r = to_np(result.factors.r)
    mask = to_np(result.sparse_mask.mask).astype(bool)
    comp = to_np(result.comp_mask.mask).astype(bool)
    a_pool = to_np(result.implicit.a_pool)
    if not ((r > 0).all() and (r <= 1.0 + tol).all()):
        return False
    implied = r + np.where(~mask & comp, a_pool, 0.0).sum(axis=1)
    if not (implied <= 1.0 + tol).all():
        return False
    if not mask.any(axis=1).all():
        return False
    return bool(np.abs(a_pool.sum(axis=1) - 1.0).max() <= tol)


def sparsity_and_flops(mask, grid: BlockGrid, d: int):
    """Sparsity ratio and dense / executed FLOPs (metrics.py:71-87)."""
    block_mask = mask.mask if hasattr(mask, "mask") else mask
    if _is_torch(block_mask):
        block_mask = block_mask.detach().cpu().numpy()
    block_mask = np.asarray(block_mask, dtype=bool)
    n, m, b = grid.n_q, grid.n_kv, grid.block
    t_v = n * b
    t = t_v + grid.t_text
    sparsity = 1.0 - int(block_mask.sum()) / (n * m)
    lens = np.asarray(grid.kv_block_lengths(), dtype=np.int64)
    flops_full = 4 * t_v * t * d
    flops_sparse = int(4 * b * d * (block_mask * lens[None, :]).sum())
    flops_overhead = sum(stage_op_counts(grid, d).values())
    return sparsity, flops_full, flops_sparse, flops_overhead


def inv_sqrt(d: int) -> float:
    return 1.0 / math.sqrt(d)
