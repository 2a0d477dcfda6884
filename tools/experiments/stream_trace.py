"""Timeline of CTA 0 of the streamed one-tile K3 experiment (kernel="tcgen05-stream";
source kept in tools/experiments/attn_stream_kernel.cu.txt, not built -- restore it into
csrc/attn_tc.cu with its RSA_KERNEL_TCGEN05_STREAM = 5 enum to rerun) at the
HunyuanVideo shape, from a tools-only -DRSA_PAIR_TRACE build:

    tools/build_variants.sh trace -DRSA_PAIR_TRACE
    RSA_B200_LIB=tools/ab_so/trace.so python tools/experiments/stream_trace.py

Per block G (cycles, medians over the CTA's blocks): the softmax halves' S
wait, S load, exps, the quad barrier, the pv_done wait and the P release, and
the MMA thread's s_free / p_full / kv waits; the block period."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2511_19835_b200 import _native as nat  # noqa: E402
from paper_2511_19835_b200.pipeline import _ptr, _stream, workspace_for  # noqa: E402

cfg = bench.CONFIGS["hv"]
dev = torch.device("cuda", 0)
heads = 24
q, k, v = bench.synth_inputs(torch, cfg, heads, 1234, dev)
shape = nat.make_shape(heads, cfg["t_v"], cfg["t_t"], 128, 128, "bfloat16", "tcgen05-stream")
conf = nat.make_config(0.1, 0.0, 0, False, "sparse-rectified")
ws = workspace_for(shape, dev)
out = torch.empty_like(q)
lib = nat.lib()
for _ in range(3):
    nat.check(lib.rsa_forward(C.byref(shape), C.byref(conf), _ptr(q), _ptr(k), _ptr(v), _ptr(out), None,
                              _ptr(ws), _stream()))
torch.cuda.synchronize()
buf = (C.c_longlong * (4 * 16384))()
assert lib.rsa_debug_pair_trace(buf, 4 * 16384) == 0
tr = np.frombuffer(buf, dtype=np.int64).reshape(4, 16384 // 8, 8)
nb = int((tr[1, :, 6] > 0).sum())
print(f"blocks traced: {nb}")
sm = tr[1, 2:nb - 1]
for h in (1, 2):
    x = tr[h, 2:nb - 1].astype(np.float64)
    per = np.diff(x[:, 1])
    sp = x[:, 3] > 0   # speculative blocks
    d = lambda a, b: np.median((x[:, b] - x[:, a])[sp])  # noqa: E731
    print(f"softmax half {h - 1}: period median {np.median(per):.0f} mean {per.mean():.0f};"
          f" S wait {np.median(x[:, 1] - x[:, 0]):.0f}, S load {d(1, 2):.0f}, exps {d(2, 3):.0f},"
          f" quad barrier {d(3, 4):.0f}, to pv_done {d(4, 5):.0f}, P store+release {d(5, 6):.0f}")
m = tr[0, 2:nb - 1].astype(np.float64)
print(f"S warp: s_free wait {np.median(m[:, 1] - m[:, 0]):.0f}, to MMA issue {np.median(m[:, 5] - m[:, 1]):.0f},"
      f" S MMAs {np.median(m[:, 6] - m[:, 5]):.0f}, after S to next {np.median(m[1:, 0] - m[:-1, 6]):.0f},"
      f" period {np.median(np.diff(m[:, 0])):.0f}")
print(f"PV warp: p_full wait {np.median(m[:, 3] - m[:, 2]):.0f}, PV MMAs {np.median(m[:, 7] - m[:, 4]):.0f},"
      f" after PV to next {np.median(m[1:, 2] - m[:-1, 7]):.0f}, period {np.median(np.diff(m[:, 2])):.0f}")
# cross: S_{G} ready (softmax S wait end) vs P_{G-2} release; pv wait
rel = tr[1, 2:nb - 1, 6].astype(np.float64)
sready = tr[1, 2:nb - 1, 1].astype(np.float64)
print(f"softmax idle between P release (G) and S_(G+1) ready: median {np.median(sready[1:] - rel[:-1]):.0f}")
# cross-warp latencies on the SM clock (block index G, rows of tr[.., G, ..])
sx = tr[1, :nb].astype(np.float64)       # softmax half 0
mx = tr[0, :nb].astype(np.float64)       # MMA thread
G = np.arange(4, nb - 2)
rel_prev = sx[G - 1, 6]                  # P_{G-1} released
print("relative to the P_{G-1} release (medians):")
print(f"  MMA sees p_full_{{G-1}}: {np.median(mx[G - 1, 3] - rel_prev):.0f};"
      f" PV_(G-1) issued: {np.median(mx[G - 1, 7] - rel_prev):.0f};"
      f" softmax G past pv_done wait: {np.median(sx[G, 5] - rel_prev):.0f};"
      f" softmax G reached pv_done wait: {np.median(sx[G, 4] - rel_prev):.0f}")
print(f"  S_G issued (MMA it. G-2, pt 6): {np.median(mx[G - 2, 6] - rel_prev):.0f};"
      f" softmax G past s_full wait: {np.median(sx[G, 1] - rel_prev):.0f}")
print(f"  S_(G+1) issued: {np.median(mx[G - 1, 6] - rel_prev):.0f}; MMA s_free_(G-1) seen: {np.median(mx[G - 1, 1] - rel_prev):.0f}")
ob = tr[3, :nb].astype(np.float64)
if ob[10, 0] > 0:
    print("observer (S_G / PV_G complete) relative to the P_{G-1} release:")
    print(f"  S_(G+1) complete: {np.median(ob[G + 1, 0] - rel_prev):.0f}; PV_(G-2) complete: {np.median(ob[G - 2, 1] - rel_prev):.0f};"
          f" PV_(G-1) complete: {np.median(ob[G - 1, 1] - rel_prev):.0f}; S_(G+2) complete: {np.median(ob[G + 2, 0] - rel_prev):.0f}")
    print(f"  PV latency (issued -> complete): {np.median(ob[G - 1, 1] - mx[G - 1, 7]):.0f};"
          f" S latency: {np.median(ob[G, 0] - mx[G - 2, 6]):.0f}")
