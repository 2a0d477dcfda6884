"""Per-tile timeline of one persistent K3 CTA (RSA_TC_STAMPS=3): step loop,
next-Q store, epilogue, gap to the next tile's first S.  HV shape, 24 heads."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("RSA_TC_PP", "0")   # the stamps are implemented in the persistent / one-tile kernels
os.environ["RSA_TC_STAMPS"] = "3"
os.environ.setdefault("RSA_TC_TRACE_CTA", "7")
import bench  # noqa: E402
from paper_2511_19835_b200 import _native as nat  # noqa: E402
from paper_2511_19835_b200.pipeline import _ptr, _stream, workspace_for  # noqa: E402

cfg = bench.CONFIGS["hv"]
dev = torch.device("cuda", 0)
heads = cfg["heads"]
q, k, v = bench.synth_inputs(torch, cfg, heads, 1234, dev)
shape = nat.make_shape(heads, cfg["t_v"], cfg["t_t"], 128, 128, "bfloat16")
conf = nat.make_config(0.1, 0.0, 0, False, "sparse-rectified")
ws = workspace_for(shape, dev)
out = torch.empty_like(q)
lse = torch.zeros(heads * q.shape[1] + 4096, dtype=torch.float32, device=dev)
for _ in range(2):
    nat.check(nat.lib().rsa_forward(C.byref(shape), C.byref(conf), _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                    _ptr(lse), _ptr(ws), _stream()))
torch.cuda.synchronize()
st = lse[:2048].view(torch.int64).view(256, 4).cpu().numpy()
L = nat.layout(shape)
vt = 928
tc = ws[L["kv_count"]:L["kv_count"] + heads * vt * 4].view(torch.int32).cpu().numpy()   # B = 128: tile = block
cta, grid, tph = int(os.environ["RSA_TC_TRACE_CTA"]), 148, 16 + vt
rows = []
for i in range(256):
    bid = cta + i * grid
    if bid >= heads * tph or st[i, 0] == 0:
        break
    h, r = divmod(bid, tph)
    count = 117 if r < 16 else int(tc[h * vt + r - 16])
    rows.append((count, *st[i]))
rows = np.array(rows, dtype=np.int64)
loop = rows[:, 2] - rows[:, 1]
qst = rows[:, 3] - rows[:, 2]
epi = rows[:, 4] - rows[:, 3]
gap = rows[1:, 1] - rows[:-1, 4]
print(f"tiles {len(rows)}; median steps {np.median(rows[:, 0])}")
print(f"cycles/step in loop: median {np.median(loop / rows[:, 0]):.0f}")
print(f"next-Q store: median {np.median(qst):.0f}; epilogue: median {np.median(epi):.0f}; "
      f"epilogue end -> next first S: median {np.median(gap):.0f}")
per_tile = np.median(np.diff(rows[:, 1]))
print(f"tile period median {per_tile:.0f} cycles; loop share {np.median(loop) / per_tile:.3f}")
