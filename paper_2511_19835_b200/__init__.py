"""B200-native Rectified SpaAttn (arXiv 2511.19835) hot path.

Drop-in for the reference package ``rectattn``'s attention entry points
(pkg/src/rectattn/__init__.py:4-24): the same containers, configuration,
variants and exceptions, backed by four hand-written sm_100a stages in
``librsa_b200.so`` (pool -> select -> block-sparse attention with the IPAR/GAPR
rectification epilogue).  There is no CPU fallback.
"""

from .core import (VARIANTS, AttentionOutput, AttentionProblem, BlockGrid, CompensationMask,
                   ImplicitAttention, PipelineAccounting, PipelineResult, PooledSet,
                   RectificationFactors, SparseMask, SparsityConfig, check_result_invariants,
                   DenominatorReport, GainError,
                   partition, sparsity_and_flops)
from .errors import (BlockSizeError, ConfigError, DegenerateRowError, EmptyRowError, IoError,
                     MissingGridError, NativeError, RectAttnError, SchemaError, ShapeError,
                     ZeroReferenceError, ZeroVectorError)

__version__ = "0.1.0"

_LAZY = {"rectified_attention_pipeline", "block_sparse_attention", "text_full_attention",
         "rectified_sparse_attention", "new_status", "raise_for_status"}
_REORDER = {"morton_permutation", "reorder_morton", "inverse_permutation"}
_DIAG = {"gain_error", "gapr_condition_agreement", "denominator_equivalence_report"}
_HARNESS = {"run_variants", "full_attention_reference", "normalized_l1", "cosine_similarity", "AlignmentReport"}
_EXPERIMENT = {"SyntheticSpec", "ExperimentConfig", "gen_synthetic", "load_problem", "save_problem",
               "run_experiment", "sweep_sparsity"}


def __getattr__(name):
    # the pipeline module imports torch; keep `import paper_2511_19835_b200` light
    if name in _LAZY:
        from . import pipeline
        return getattr(pipeline, name)
    if name in _REORDER:
        from . import reorder
        return getattr(reorder, name)
    if name in _DIAG:
        from . import diagnostics
        return getattr(diagnostics, name)
    if name in _HARNESS:
        from . import harness
        return getattr(harness, name)
    if name in _EXPERIMENT:
        from . import experiment
        return getattr(experiment, name)
    raise AttributeError(name)
