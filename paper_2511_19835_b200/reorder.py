"""Morton (Z-order) token reordering (reference core.py:263-325) and the
permuted-problem entry point.

* ``morton_permutation(grid_dims)``: ``rsa_morton_permutation`` in the library
  (host: Morton codes, stable sort -- numpy's ``argsort(kind="stable")``).
* ``reorder_morton(problem)``: the reordered problem and the permutation, like
  the reference (core.py:294-318); the row moves run on the GPU
  (``rsa_permute_rows``).
* ``inverse_permutation(perm)``: core.py:321-325 (index bookkeeping).
* ``rectified_sparse_attention(..., grid_dims=..., morton=True)``: the
  reference harness's ``morton_reorder`` pipeline (harness.py:172-173) fused
  into K1 (row gather) and the K3 epilogue (row scatter): inputs and outputs
  in the original token order (``rsa_forward_permuted``).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .core import AttentionProblem, _is_torch
from .errors import MissingGridError, ShapeError

_PERM_CACHE: dict = {}


def morton_permutation(grid_dims) -> np.ndarray:
    """Permutation ``p`` such that ``tokens[p]`` is in 3-D Morton order over
    (t, h, w), w fastest. core.py:276-291."""
    t, h, w = (int(x) for x in grid_dims)
    out = np.empty(t * h * w, dtype=np.int32)
    nat.check(nat.lib().rsa_morton_permutation(t, h, w, out.ctypes.data_as(C.c_void_p)))
    return out.astype(np.int64)


def inverse_permutation(perm) -> np.ndarray:
    """core.py:321-325."""
    perm = np.asarray(perm)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    return inv


def device_permutation(grid_dims, device):
    """The Morton permutation as a cached device int32 tensor (K1/K3 operand)."""
    import torch
    key = (tuple(int(x) for x in grid_dims), str(device))
    p = _PERM_CACHE.get(key)
    if p is None:
        p = torch.from_numpy(morton_permutation(grid_dims).astype(np.int32)).to(device)
        _PERM_CACHE[key] = p
    return p


def _permute(x, t_v, t_t, perm_dev, inverse=False):
    """Rows [0, t_v) of x permuted on the GPU (rsa_permute_rows); rows after
    them copied.  numpy in -> numpy out, torch in -> torch out."""
    import torch

    from .pipeline import _as_tensor, _device, _ptr, _stream
    host = not _is_torch(x)
    dev = _device()
    xt = _as_tensor(x, dev).contiguous()
    out = torch.empty_like(xt)
    shape = nat.make_shape(1, t_v, t_t, xt.shape[1], 1, str(xt.dtype).replace("torch.", ""))
    nat.check(nat.lib().rsa_permute_rows(C.byref(shape), _ptr(perm_dev), _ptr(xt), _ptr(out),
                                         1 if inverse else 0, _stream()))
    if host:
        return out.cpu().numpy()
    return out


def reorder_morton(problem: AttentionProblem):
    """Permute the video tokens of Q/K/V into Morton order over (t, h, w);
    text rows untouched.  Returns ``(reordered_problem, permutation)`` with
    ``permutation[i]`` the original row now at video row ``i``. core.py:294-318."""
    if problem.grid_dims is None:
        raise MissingGridError("reorder_morton needs grid_dims on the problem")
    from .pipeline import _device
    perm = morton_permutation(problem.grid_dims)
    perm_dev = device_permutation(problem.grid_dims, _device())
    t_v, t_t = problem.t_v, problem.t_t
    reordered = AttentionProblem(
        q_video=_permute(problem.q_video, t_v, 0, perm_dev),
        q_text=problem.q_text.copy() if not _is_torch(problem.q_text) else problem.q_text.clone(),
        k=_permute(problem.k, t_v, t_t, perm_dev),
        v=_permute(problem.v, t_v, t_t, perm_dev),
        d=problem.d, block=problem.block, grid_dims=problem.grid_dims)
    return reordered, perm


def permuted_forward(q, k, v, shape, cfg, perm_dev, lse, workspace):
    """rsa_forward_permuted on [heads, T, d]-contiguous CUDA tensors."""
    import torch

    from .pipeline import _ptr, _stream, workspace_for
    if perm_dev.numel() != shape.t_video:
        raise ShapeError(f"permutation has {perm_dev.numel()} entries, T_v = {shape.t_video}")
    size = nat.lib().rsa_permuted_buffer_size(C.byref(shape))
    perm_buf = torch.empty(size, dtype=torch.uint8, device=q.device)
    if workspace is None:
        workspace = workspace_for(shape, q.device)
    out = torch.empty_like(q)
    nat.check(nat.lib().rsa_forward_permuted(C.byref(shape), C.byref(cfg), _ptr(q), _ptr(k), _ptr(v),
                                             _ptr(perm_dev), _ptr(perm_buf), _ptr(out), _ptr(lse),
                                             _ptr(workspace), _stream()))
    return out
