"""The drop-in entry points: the reference's pipeline / kernel API backed by
librsa_b200.so, plus the batched tensor op a model integration calls.

Reference entry points mirrored here (pkg/src/rectattn):
  rectified_attention_pipeline(problem, config, variant)   rectify.py:107-176
  block_sparse_attention(q_v, k, v, mask, grid, counters)  kernel.py:65-117
  text_full_attention(q_t, k, v, block)                    kernel.py:120-145
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as nat
from .core import (VARIANTS, AttentionOutput, AttentionProblem, BlockGrid, CompensationMask,
                   ImplicitAttention, PipelineAccounting, PipelineResult, PooledSet,
                   RectificationFactors, SparseMask, SparsityConfig, _is_torch, check_matrix,
                   partition, stage_op_counts)
from .errors import ConfigError, EmptyRowError, NativeError, ShapeError

MASK_BIT, IMPORTANCE_BIT, COMP_BIT, ADJ_BIT, APPLIED_BIT = 1, 2, 4, 8, 16


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the B200 kernels are the only implementation "
                          "(there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _as_tensor(x, device) -> torch.Tensor:
    if _is_torch(x):
        return x.to(device)
    return torch.from_numpy(np.ascontiguousarray(x)).to(device)


def _promote(device, *xs) -> list:
    """Device copies of q/k/v in their common dtype -- numpy's promotion of
    mixed-precision operands in kernel.py (float32 with float64 computes in
    float64); the kernels read all three buffers in one dtype."""
    ts = [_as_tensor(x, device) for x in xs]
    dt = ts[0].dtype
    for t in ts[1:]:
        dt = torch.promote_types(dt, t.dtype)
    return [t.to(dt).contiguous() for t in ts]


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def workspace_for(shape: nat.Shape, device) -> torch.Tensor:
    size = nat.lib().rsa_workspace_size(C.byref(shape))
    if size == 0:
        nat.check(nat.lib().rsa_plan(C.byref(shape), None, None))
    return torch.empty(size, dtype=torch.uint8, device=device)


def _checked_workspace(workspace, shape: nat.Shape, device) -> torch.Tensor:
    """The caller's workspace, checked against this shape (a workspace sized for
    a smaller problem would be overrun on the device), or a fresh one."""
    if workspace is None:
        return workspace_for(shape, device)
    need = nat.lib().rsa_workspace_size(C.byref(shape))
    if workspace.device != device or workspace.numel() * workspace.element_size() < need:
        raise ShapeError(f"workspace holds {workspace.numel() * workspace.element_size()} bytes on "
                         f"{workspace.device}; this shape needs {need} bytes on {device}")
    if not workspace.is_contiguous():
        raise ShapeError("workspace must be contiguous")
    return workspace


def _check_lse(lse, rows: int, device) -> None:
    if lse is None:
        return
    if lse.dtype != torch.float32 or lse.numel() < rows or not lse.is_contiguous():
        raise ShapeError(f"lse must be a contiguous float32 tensor of >= {rows} entries, "
                         f"got {lse.dtype} with {lse.numel()}")
    if device.type == "cuda" and lse.device != device:
        raise ShapeError(f"lse is on {lse.device}, inputs on {device}")


def _view(ws: torch.Tensor, offset: int, dtype, shape) -> torch.Tensor:
    n = int(np.prod(shape))
    itemsize = torch.empty((), dtype=dtype).element_size()
    return ws[offset:offset + n * itemsize].view(dtype).view(*shape)


def _cfg_tuple(config) -> tuple:
    return (config.top_k_fraction, config.weight_threshold, config.adjacency_radius,
            config.force_text_blocks)


# ---------------------------------------------------------------------------
# rectify.py:107-176
# ---------------------------------------------------------------------------

def rectified_attention_pipeline(problem: AttentionProblem, config: SparsityConfig,
                                 variant: str = "sparse-rectified", *, kernel: str = "auto",
                                 timing: bool = False) -> PipelineResult:
    """Pool, implicit full attention, gain/error and compensation mask, sparse
    mask, sparse kernel plus text full attention, then the variant's
    rectification step -- all on the GPU (K1 -> K2 -> K3+K4)."""
    if variant not in VARIANTS:
        raise ConfigError(f"unknown variant {variant!r}, expected one of {VARIANTS}")
    dev = _device()
    host = not _is_torch(problem.q_video)
    grid = partition(problem)
    t_v, t_t, d = problem.t_v, problem.t_t, problem.d
    q = torch.cat([_as_tensor(problem.q_video, dev), _as_tensor(problem.q_text, dev)]).contiguous()
    k = _as_tensor(problem.k, dev).contiguous()
    v = _as_tensor(problem.v, dev).contiguous()
    dtype = str(q.dtype).replace("torch.", "")
    shape = nat.make_shape(1, t_v, t_t, d, problem.block, dtype, kernel, ragged_video=grid.ragged)
    cfg = nat.make_config(*_cfg_tuple(config), variant)
    nat.plan(shape, cfg)
    ws = workspace_for(shape, dev)
    out = torch.empty_like(q)
    lse = torch.empty(q.shape[0], dtype=torch.float32, device=dev)
    lib, st = nat.lib(), _stream()
    acct = PipelineAccounting()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timing else None
    if ev:
        ev[0].record()
    nat.check(lib.rsa_pool(C.byref(shape), _ptr(q), _ptr(k), _ptr(v), _ptr(ws), st))
    if ev:
        ev[1].record()
    nat.check(lib.rsa_select(C.byref(shape), C.byref(cfg), _ptr(ws), st))
    if ev:
        ev[2].record()
    nat.check(lib.rsa_attention(C.byref(shape), C.byref(cfg), _ptr(q), _ptr(k), _ptr(v),
                                _ptr(out), _ptr(lse), _ptr(ws), st))
    if ev:
        ev[3].record()
    nat.check(lib.rsa_check_device_status(_ptr(ws), st))  # synchronises (reference raises eagerly)
    if ev:
        acct.stage_wall_ms = {"pool": ev[0].elapsed_time(ev[1]),
                              "select": ev[1].elapsed_time(ev[2]),
                              "attention": ev[2].elapsed_time(ev[3])}
    return _result(problem, grid, shape, ws, out, lse, variant, acct, host)


def _result(problem, grid: BlockGrid, shape, ws, out, lse, variant, acct, host) -> PipelineResult:
    L = nat.layout(shape)
    N, M, d, t_v, t_t = grid.n_q, grid.n_kv, problem.d, problem.t_v, problem.t_t
    n_cols = N + t_t + (M - N)
    f64 = torch.float64
    q_pool = _view(ws, L["q_pool"], f64, (N, d))
    k_cat = _view(ws, L["k_cat"], f64, (n_cols, d))
    v_pool = _view(ws, L["v_pool"], f64, (M, d))
    scores = _view(ws, L["scores"], f64, (N, n_cols))
    a_pool = _view(ws, L["a_pool"], f64, (N, M))
    bits = _view(ws, L["mask_bits"], torch.uint8, (N, M))
    r = _view(ws, L["r"], f64, (N,))
    mask = (bits & MASK_BIT) != 0
    conv = (lambda x: x.detach().cpu().numpy()) if host else (lambda x: x.clone())
    lens = torch.tensor(grid.kv_block_lengths(), dtype=torch.int64, device=bits.device)
    qlens = torch.tensor(grid.q_block_lengths(), dtype=torch.int64, device=bits.device)
    acct.kernel_inner_product_ops = int((mask.to(torch.int64) * lens[None, :] * qlens[:, None]).sum().item()) * d
    acct.stage_ops = stage_op_counts(grid, d)
    out_dtype = problem.q_video.dtype
    o = conv(out)
    o_video, o_text = o[:t_v], o[t_v:]
    if host:
        o_video, o_text = o_video.astype(out_dtype), o_text.astype(out_dtype)
    return PipelineResult(
        output=AttentionOutput(o_video=o_video, o_text=o_text,
                               row_log_denominators=conv(lse[:t_v].to(f64))),
        factors=RectificationFactors(r=conv(r)),
        implicit=ImplicitAttention(conv(a_pool), scores[:, :N + t_t].clone(), N, grid.block, t_t, conv),
        sparse_mask=SparseMask(mask=conv(mask), importance=conv((bits & IMPORTANCE_BIT) != 0),
                               adjacency=conv((bits & ADJ_BIT) != 0),
                               retained_count=conv(mask.sum(dim=1))),
        comp_mask=CompensationMask(mask=conv((bits & COMP_BIT) != 0)),
        accounting=acct, grid=grid,
        pooled=PooledSet(q_pool=conv(q_pool), k_v_pool=conv(k_cat[:N]), v_pool=conv(v_pool),
                         k_mix_pool=conv(k_cat[:N + t_t])),
        variant=variant)


# ---------------------------------------------------------------------------
# kernel.py:65-117 and kernel.py:120-145
# ---------------------------------------------------------------------------

def block_sparse_attention(q_v, k, v, mask, grid: BlockGrid, counters: dict | None = None,
                           *, kernel: str = "auto"):
    """Sparse attention of the video queries over an explicit (N, M) block mask.
    Returns ``(o_video, row_log_denominators)``."""
    check_matrix(q_v, "q_v")
    check_matrix(k, "k")
    check_matrix(v, "v")
    block_mask = getattr(mask, "mask", mask)
    host = not _is_torch(q_v)
    dev = _device()
    bm = _as_tensor(np.asarray(block_mask, dtype=bool) if not _is_torch(block_mask) else block_mask,
                    dev).to(torch.bool)
    if tuple(bm.shape) != (grid.n_q, grid.n_kv):
        raise ShapeError(f"mask shape {tuple(bm.shape)} != (N, M) = {(grid.n_q, grid.n_kv)}")
    if q_v.shape[0] != grid.t_video:
        raise ShapeError(f"q_v has {q_v.shape[0]} rows, expected {grid.t_video} (the grid's video tokens)")
    if tuple(k.shape) != tuple(v.shape):
        raise ShapeError(f"k shape {tuple(k.shape)} != v shape {tuple(v.shape)}")
    if k.shape[0] != grid.t_video + grid.t_text or k.shape[1] != q_v.shape[1]:
        raise ShapeError(f"k has shape {tuple(k.shape)}, expected ({grid.t_video + grid.t_text}, "
                         f"{q_v.shape[1]}) (video + text tokens of the grid, head_dim of q_v)")
    empty = ~bm.any(dim=1)
    if bool(empty.any()):
        raise EmptyRowError(f"mask rows {torch.nonzero(empty).flatten().tolist()} retain no key block")
    t_v, d = q_v.shape[0], q_v.shape[1]
    t_t = k.shape[0] - t_v
    qv, kk, vv = _promote(dev, q_v, k, v)
    q = torch.cat([qv, torch.zeros(t_t, d, dtype=qv.dtype, device=dev)]).contiguous()
    shape = nat.make_shape(1, t_v, t_t, d, grid.block, str(q.dtype).replace("torch.", ""), kernel,
                           ragged_video=grid.ragged)
    ws = workspace_for(shape, dev)
    out = torch.zeros_like(q)
    lse = torch.empty(q.shape[0], dtype=torch.float32, device=dev)
    m8 = bm.to(torch.uint8).contiguous()
    nat.check(nat.lib().rsa_block_sparse_attention(C.byref(shape), _ptr(q), _ptr(kk), _ptr(vv),
                                                   _ptr(m8), _ptr(out), _ptr(lse), _ptr(ws), _stream()))
    nat.check(nat.lib().rsa_check_device_status(_ptr(ws), _stream()))
    if counters is not None:
        lens = torch.tensor(grid.kv_block_lengths(), dtype=torch.int64, device=dev)
        qlens = torch.tensor(grid.q_block_lengths(), dtype=torch.int64, device=dev)
        ops = int((bm.to(torch.int64) * lens[None, :] * qlens[:, None]).sum().item()) * d
        counters["inner_product_ops"] = counters.get("inner_product_ops", 0) + ops
    o_video, ld = out[:t_v], lse[:t_v].to(torch.float64)
    if host:
        return o_video.cpu().numpy(), ld.cpu().numpy()
    return o_video, ld


def text_full_attention(q_t, k, v, block: int = 128):
    """Full attention for text queries over every key, tiled by ``block``."""
    check_matrix(q_t, "q_t")
    check_matrix(k, "k")
    check_matrix(v, "v")
    if q_t.shape[1] != k.shape[1]:
        raise ShapeError(f"q_t width {q_t.shape[1]} != k width {k.shape[1]}")
    if tuple(k.shape) != tuple(v.shape):
        raise ShapeError(f"k shape {tuple(k.shape)} != v shape {tuple(v.shape)}")
    host = not _is_torch(q_t)
    if q_t.shape[0] == 0:
        return (np.empty((0, v.shape[1]), dtype=q_t.dtype) if host
                else torch.empty(0, v.shape[1], dtype=q_t.dtype, device=q_t.device))
    dev = _device()
    q, kk, vv = _promote(dev, q_t, k, v)
    out = torch.empty_like(q)
    code = nat.DTYPE_CODES[str(q.dtype).replace("torch.", "")]
    nat.check(nat.lib().rsa_text_full_attention(1, q.shape[0], kk.shape[0], q.shape[1], int(block),
                                                code, _ptr(q), _ptr(kk), _ptr(vv), _ptr(out), None,
                                                None, _stream()))
    if host:
        return out.cpu().numpy()
    return out


# ---------------------------------------------------------------------------
# batched tensor op: [batch, heads, T, d] (video tokens first)
# ---------------------------------------------------------------------------

def rectified_sparse_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *,
                               num_text_tokens: int, block: int = 128,
                               top_k_fraction: float | None = None,
                               weight_threshold: float = 0.0, adjacency_radius: int = 0,
                               force_text_blocks: bool = False,
                               variant: str = "sparse-rectified", sparsity: float | None = None,
                               kernel: str = "auto", lse: torch.Tensor | None = None,
                               workspace: torch.Tensor | None = None,
                               check_status: bool = True, status: torch.Tensor | None = None,
                               heads_per_chunk: int = 1,
                               grid_dims: tuple | None = None, morton: bool = False,
                               ragged_video: bool = False, out: torch.Tensor | None = None) -> torch.Tensor:
    """Rectified block-sparse attention for every (batch, head) of q/k/v
    ([..., T, d], the last ``num_text_tokens`` rows text).  ``sparsity=s`` is
    shorthand for top_k_fraction = 1 - s with p = 0, r = 0, no forced text.
    Errors are the reference's exceptions (errors.py).  Shape / config errors
    raise before any launch; the device-side ones (non-finite input ->
    ShapeError, degenerate reallocation row -> DegenerateRowError, empty mask
    row -> EmptyRowError; core.py:23-31, ipar.py:62-64, kernel.py:85-87) are
    raised eagerly like the reference does when ``check_status`` (default),
    which synchronises the stream once per call.  A model loop that must not
    synchronise passes ``check_status=False`` and a zeroed int32[4] CUDA tensor
    ``status``: every call ORs its flags into it on the stream (no sync), and
    ``raise_for_status(status)`` raises the first error at the caller's next
    synchronisation point.  Host tensors (the end-to-end call): the copies in
    and out are pipelined with the compute over chunks of ``heads_per_chunk``
    heads (rsa_forward_host), the flags of every chunk are kept, checked after
    the final synchronisation, and the host output is returned.
    ``morton=True`` (needs ``grid_dims`` = (t, h, w) of the video tokens):
    the pipeline runs on the Morton-reordered problem, as the reference
    harness's ``morton_reorder`` option does (harness.py:172-173), with the
    gather fused into K1 and the scatter into the K3 epilogue -- inputs and
    output stay in the original token order.
    ``ragged_video=True`` accepts a video token count that is not a multiple of
    ``block`` (the final video block is shorter; an extension -- the reference
    raises BlockSizeError), e.g. HunyuanVideo's exact 118,800 tokens.
    ``out`` (CUDA tensors): a contiguous tensor of q's shape and dtype the
    result is written into (e.g. a slice of a caller's buffer)."""
    if sparsity is not None:
        top_k_fraction, weight_threshold, adjacency_radius, force_text_blocks = 1.0 - sparsity, 0.0, 0, False
    if top_k_fraction is None:
        top_k_fraction = 0.1
    if q.dim() < 3 or q.shape != k.shape or k.shape != v.shape:
        raise ShapeError(f"q/k/v must share a [..., T, d] shape, got {tuple(q.shape)}, "
                         f"{tuple(k.shape)}, {tuple(v.shape)}")
    T, d = q.shape[-2], q.shape[-1]
    heads = int(np.prod(q.shape[:-2]))
    t_t = int(num_text_tokens)
    shape = nat.make_shape(heads, T - t_t, t_t, d, block, str(q.dtype).replace("torch.", ""), kernel,
                           ragged_video=ragged_video)
    cfg = nat.make_config(top_k_fraction, weight_threshold, adjacency_radius, force_text_blocks, variant)
    nat.plan(shape, cfg)
    if not q.is_cuda:
        if morton:
            raise ShapeError("morton=True needs CUDA tensors (use reorder_morton for host arrays)")
        if k.is_cuda or v.is_cuda:
            raise ShapeError("q, k and v must all be host tensors or all CUDA tensors")
        return _forward_from_host(q, k, v, shape, cfg, lse, workspace, heads_per_chunk, status)
    strided = _strided_layout(q, k, v, kernel, morton)
    if strided is None:
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    workspace = _checked_workspace(workspace, shape, q.device)
    _check_lse(lse, heads * T, q.device)
    if strided is not None:
        # row-contiguous views ([B, T, H, d] transposed to [B, H, T, d], head
        # slices of a fused qkv buffer, ...) go straight to the kernels through
        # their strides: no copy.  The output keeps q's dimension order (dense).
        if out is None:
            out = _dense_like(q)
        if out.shape != q.shape or out.dtype != q.dtype or out.device != q.device:
            raise ShapeError(f"out must be a {q.dtype} tensor of shape {tuple(q.shape)} on {q.device}")
        out_layout = _layout_of(out)
        if out_layout is None:
            raise ShapeError("out must have rows of d contiguous elements at 16-byte aligned strides")
        nat.check(nat.lib().rsa_forward_strided(C.byref(shape), C.byref(cfg), C.byref(strided), C.byref(out_layout),
                                                _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), _ptr(workspace),
                                                _stream()))
    elif morton:
        from .errors import MissingGridError
        from .reorder import device_permutation, permuted_forward
        if grid_dims is None:
            raise MissingGridError("morton=True needs grid_dims")
        t, hh, w = grid_dims
        if t * hh * w != T - t_t:
            raise ShapeError(f"grid_dims product {t * hh * w} != T_v={T - t_t}")
        if out is not None:
            raise ShapeError("out= is not supported with morton=True")
        out = permuted_forward(q, k, v, shape, cfg, device_permutation(grid_dims, q.device), lse, workspace)
    else:
        if out is None:
            out = torch.empty_like(q)
        elif out.shape != q.shape or out.dtype != q.dtype or out.device != q.device or not out.is_contiguous():
            raise ShapeError(f"out must be a contiguous {q.dtype} tensor of shape {tuple(q.shape)} on {q.device}")
        nat.check(nat.lib().rsa_forward(C.byref(shape), C.byref(cfg), _ptr(q), _ptr(k), _ptr(v),
                                        _ptr(out), _ptr(lse), _ptr(workspace), _stream()))
    _report_status(workspace, status, check_status)
    return out


def _layout_of(x: torch.Tensor):
    """rsa_layout of a [..., T, d] view (up to 4-D) whose rows are contiguous
    and whose token / head / batch strides are multiples of 8 elements (16-byte
    TMA rows), else None."""
    if x.dim() > 4 or x.stride(-1) != 1 or x.data_ptr() % 16:
        return None
    st, shp = list(x.stride()), list(x.shape)
    while len(shp) < 4:
        shp.insert(0, 1)
        st.insert(0, 0)
    B, H, T = shp[0], shp[1], shp[2]
    # (a size-1 dimension's stride is never used: give it a dense value)
    tok = st[2]
    head = st[1] if H > 1 else tok * T
    bat = st[0] if B > 1 else head * H
    if tok % 8 or head % 8 or bat % 8 or head == 0 or bat == 0:   # (broadcast dims: copy instead)
        return None
    return nat.TensorLayout(int(H), int(tok), int(head), int(bat))


def _strided_layout(q, k, v, kernel, morton):
    """An rsa_layout for non-contiguous bf16 CUDA q/k/v of one shared stride
    pattern with contiguous rows -- e.g. the model's [B, T, H, d] projection
    output viewed as [B, H, T, d].  None: the contiguous path (copying if
    needed)."""
    if q.is_contiguous() and k.is_contiguous() and v.is_contiguous():
        return None
    if morton or kernel == "simt" or q.dtype != torch.bfloat16 or not (q.stride() == k.stride() == v.stride()):
        return None
    if any(x.data_ptr() % 16 for x in (k, v)):
        return None
    return _layout_of(q)


def _dense_like(x: torch.Tensor) -> torch.Tensor:
    """A dense tensor of x's shape whose dimensions are laid out in x's stride
    order (empty_like does that only for dense x): the output of a
    [B, T, 3, H, d] fused-qkv slice is a dense [B, T, H, d] buffer."""
    order = sorted(range(x.dim()), key=lambda i: (-x.stride(i), i))
    buf = torch.empty([x.shape[i] for i in order], dtype=x.dtype, device=x.device)
    inv = [order.index(i) for i in range(x.dim())]
    return buf.permute(inv)


def _report_status(workspace: torch.Tensor, status: torch.Tensor | None, check: bool) -> None:
    if status is not None:
        if status.dtype != torch.int32 or status.numel() < 4 or status.device != workspace.device:
            raise ShapeError("status must be an int32 CUDA tensor of 4 entries on the inputs' device")
        nat.check(nat.lib().rsa_accumulate_status(_ptr(workspace), _ptr(status), _stream()))
    if check:
        nat.check(nat.lib().rsa_check_device_status(_ptr(workspace), _stream()))


def new_status(device=None) -> torch.Tensor:
    """A zeroed status accumulator for ``rectified_sparse_attention(status=...)``."""
    return torch.zeros(4, dtype=torch.int32, device=device if device is not None else _device())


def raise_for_status(status: torch.Tensor) -> None:
    """Raise the reference exception for the flags accumulated in ``status``
    (synchronises with the stream that last wrote it)."""
    flags = status.detach().to("cpu", torch.int32).contiguous()
    nat.check(nat.lib().rsa_status_from_flags(_ptr(flags)))


_STAGING: dict = {}


def _forward_from_host(q, k, v, shape, cfg, lse, workspace, heads_per_chunk, status=None):
    """Host tensors in, host tensor out: rsa_forward_host pipelines the
    host->device copies, the three kernels and the device->host copy over
    chunks of heads.  Inputs should be page-locked (``pin_memory()``) for the
    copies to overlap the compute; the staging buffers are cached per shape."""
    dev = _device()
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device (there is no CPU fallback)")
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    key = (tuple(q.shape), q.dtype, dev.index)
    bufs = _STAGING.get(key)
    if bufs is None:
        _STAGING.clear()
        bufs = [torch.empty(q.shape, dtype=q.dtype, device=dev) for _ in range(4)]
        _STAGING[key] = bufs
    dq, dk, dv, dout = bufs[:4]
    if workspace is None:
        if len(bufs) == 4:
            bufs.append(workspace_for(shape, dev))
        workspace = bufs[4]
    workspace = _checked_workspace(workspace, shape, dev)
    _check_lse(lse, int(np.prod(q.shape[:-1])), dev)
    out = torch.empty(q.shape, dtype=q.dtype, pin_memory=q.is_pinned())
    nat.check(nat.lib().rsa_forward_host(C.byref(shape), C.byref(cfg), _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                         _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dout), _ptr(lse),
                                         _ptr(workspace), int(heads_per_chunk), _stream()))
    # flags of every head chunk (rsa_forward_host clears them once); synchronises
    _report_status(workspace, status, True)
    return out
