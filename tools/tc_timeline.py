"""Per-CTA timeline of the tcgen05 kernel at the HV shape (RSA_TC_MODE=7 stamps)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("RSA_TC_PP", "0")   # the stamps are implemented in the persistent / one-tile kernels
os.environ["RSA_TC_STAMPS"] = "1"
import bench  # noqa: E402
from paper_2511_19835_b200 import _native as nat  # noqa: E402
from paper_2511_19835_b200.pipeline import _ptr, _stream, workspace_for  # noqa: E402

cfg = bench.CONFIGS["hv"]
dev = torch.device("cuda", 0)
heads = int(sys.argv[1]) if len(sys.argv) > 1 else 24
q, k, v = bench.synth_inputs(torch, cfg, heads, 1234, dev)
shape = nat.make_shape(heads, cfg["t_v"], cfg["t_t"], 128, 128, "bfloat16")
conf = nat.make_config(0.1, 0.0, 0, False, "sparse-rectified")
ws = workspace_for(shape, dev)
out = torch.empty_like(q)
lse = torch.zeros(heads * q.shape[1] * 2 + (1 << 20), dtype=torch.float32, device=dev)
lib = nat.lib()
for _ in range(2):
    nat.check(lib.rsa_forward(C.byref(shape), C.byref(conf), _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse),
                              _ptr(ws), _stream()))
torch.cuda.synchronize()
tph = 2 * 8 + 928   # per head: 2 text tiles x 8 split-K chunks, then 928 video tiles
tiles = heads * tph
ts = lse.view(torch.int64)[:tiles * 8].view(tiles, 8).cpu().numpy()
is_vid = (np.arange(tiles) % tph) >= 16
t0 = ts[:, 0].min()
rel = (ts[:, :7] - t0) / 1e3  # us
vid = rel[is_vid]
print("kernel span us", rel[:, 6].max())
for name, a, b in [("setup", 0, 1), ("q->first mma (mma thread)", 1, 2), ("mma loop", 2, 3),
                   ("softmax end - mma end", 3, 4), ("epilogue", 4, 5), ("teardown wait", 5, 6), ("total", 0, 6)]:
    dd = vid[:, b] - vid[:, a]
    print(f"{name:28s} median {np.median(dd):8.2f} us  p90 {np.percentile(dd, 90):8.2f}")
tsv = ts[is_vid]
sm = tsv[:, 7]
# gap between consecutive CTAs on the same SM
gaps = []
for s_ in np.unique(sm)[:148]:
    idx = np.where(sm == s_)[0]
    st = np.sort(tsv[idx, 0])
    en = np.sort(tsv[idx, 6])
    if len(st) > 2:
        gaps.extend(((st[1:] - en[:-1]) / 1e3).tolist())
print("launch gap between CTAs on one SM: median %.2f us p90 %.2f" % (np.median(gaps), np.percentile(gaps, 90)))
steps = ws  # noqa
