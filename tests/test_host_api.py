"""Host-side containers and validation of the reference surface (no GPU)."""

import numpy as np
import pytest

import paper_2511_19835_b200 as rsa
from paper_2511_19835_b200 import (AttentionProblem, BlockSizeError, ConfigError, ShapeError,
                                   SparsityConfig, partition)
from oracle import rsa_oracle as O


def problem(t_v=8, t_t=3, d=8, block=4, dtype=np.float64, **kw):
    qv, qt, k, v = O.random_problem(0, t_v=t_v, t_t=t_t, d=d, dtype=dtype)
    return AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=d, block=block, **kw)


def test_partition_ragged_text():
    g = partition(problem(8, 3, 8, 4))
    assert (g.n_q, g.n_kv, g.last_text_block_len) == (2, 3, 3)
    assert g.kv_block_lengths() == [4, 4, 3]
    assert g.t_text == 3


def test_problem_validation():
    with pytest.raises(BlockSizeError):
        problem(7, 0, 8, 4)
    with pytest.raises(BlockSizeError):
        problem(8, 0, 8, 0)
    qv, qt, k, v = O.random_problem(0, t_v=8, t_t=2, d=8)
    with pytest.raises(ShapeError):
        AttentionProblem(q_video=qv, q_text=qt, k=k[:-1], v=v, d=8, block=4)
    with pytest.raises(ShapeError):
        AttentionProblem(q_video=qv.astype(np.float32), q_text=qt, k=k, v=v, d=8, block=4)
    bad = qv.copy()
    bad[0, 0] = np.nan
    with pytest.raises(ShapeError):
        AttentionProblem(q_video=bad, q_text=qt, k=k, v=v, d=8, block=4)
    with pytest.raises(ShapeError):
        problem(grid_dims=(1, 2, 3))


def test_sparsity_config_validation():
    with pytest.raises(ConfigError):
        SparsityConfig(top_k_fraction=0.0)
    with pytest.raises(ConfigError):
        SparsityConfig(weight_threshold=1.5)
    with pytest.raises(ConfigError):
        SparsityConfig(adjacency_radius=-1)
    c = SparsityConfig.from_sparsity(0.9)
    assert c.top_k_fraction == pytest.approx(0.1) and c.weight_threshold == 0.0
    assert c.adjacency_radius == 0 and not c.force_text_blocks


def test_torch_bf16_problem_accepted():
    torch = pytest.importorskip("torch")
    qv = torch.randn(8, 8, dtype=torch.bfloat16)
    qt = torch.randn(3, 8, dtype=torch.bfloat16)
    k = torch.randn(11, 8, dtype=torch.bfloat16)
    p = AttentionProblem(q_video=qv, q_text=qt, k=k, v=k.clone(), d=8, block=4)
    assert p.t_v == 8 and p.t_t == 3


def test_variants_and_exports():
    assert rsa.VARIANTS == O.VARIANTS
    for name in ("rectified_attention_pipeline", "block_sparse_attention", "text_full_attention",
                 "rectified_sparse_attention"):
        assert callable(getattr(rsa, name))


def test_sparsity_and_flops_convention():
    g = partition(problem(8, 3, 8, 4))
    mask = np.ones((g.n_q, g.n_kv), dtype=bool)
    sp, full, sparse, over = rsa.sparsity_and_flops(mask, g, 8)
    assert sp == 0.0 and full == sparse == 4 * 8 * 11 * 8 and over > 0
