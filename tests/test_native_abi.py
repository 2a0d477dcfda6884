"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and the host-side validation (no GPU needed) raises the
reference's exception classes."""

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2511_19835_b200 import _native as nat
from paper_2511_19835_b200.errors import (BlockSizeError, ConfigError, NativeError, ShapeError)

HEADER = Path(__file__).resolve().parent.parent / "include" / "rsa_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(rsa_[a-z_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = nat.lib()
    syms = declared_symbols()
    assert "rsa_forward" in syms and len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(nat.EXPORTS)


def test_version_string():
    assert "sm_100a" in nat.version()


def test_plan_grid_matches_partition():
    # core.py:140-151: N = T_v/B, M = N + ceil(T_t/B), ragged last text block
    g = nat.plan(nat.make_shape(2, 3840, 256, 64, 64, "bfloat16"),
                 nat.make_config(0.1, 0.0, 0, False, "sparse-rectified"))
    assert (g.n_q, g.n_kv, g.n_text_blocks, g.last_text_block_len) == (60, 64, 4, 64)
    g = nat.plan(nat.make_shape(1, 8, 3, 8, 4, "float64"))
    assert (g.n_q, g.n_kv, g.last_text_block_len, g.n_cols) == (2, 3, 3, 2 + 3 + 1)
    g = nat.plan(nat.make_shape(1, 8, 0, 8, 4, "float32"))
    assert (g.n_q, g.n_kv, g.last_text_block_len) == (2, 2, 0)


@pytest.mark.parametrize("t_v,block", [(7, 4), (8, 0), (8, -2)])
def test_block_size_errors(t_v, block):
    with pytest.raises(BlockSizeError):
        nat.plan(nat.make_shape(1, t_v, 0, 8, block, "float32"))


@pytest.mark.parametrize("f,p,r", [(0.0, 0.3, 1), (1.5, 0.3, 1), (0.2, -0.1, 1), (0.2, 1.5, 1), (0.2, 0.3, -1)])
def test_config_errors(f, p, r):
    with pytest.raises(ConfigError):
        nat.plan(nat.make_shape(1, 8, 0, 8, 4, "float32"), nat.make_config(f, p, r, True, "full"))


def test_unknown_variant():
    with pytest.raises(ConfigError):
        nat.make_config(0.2, 0.3, 1, True, "bogus")


def test_bad_dtype():
    with pytest.raises(ShapeError):
        nat.make_shape(1, 8, 0, 8, 4, "float16")


def test_unsupported_head_dim():
    with pytest.raises(NativeError):
        nat.plan(nat.make_shape(1, 8, 0, 512, 4, "bfloat16"))


def test_workspace_layout_is_ordered_and_aligned():
    L = nat.layout(nat.make_shape(24, 118784, 256, 128, 128, "bfloat16"))
    offs = [L[n] for n in nat.LAYOUT_FIELDS if n != "total"]
    assert all(o % 256 == 0 for o in offs)
    assert L["total"] > max(offs)
    # HunyuanVideo shape fits comfortably in 180 GB of HBM
    assert L["total"] < 2 * 1024 ** 3
