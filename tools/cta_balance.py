"""Per-CTA start/end of the persistent K3 kernel (RSA_TC_STAMPS=4): load balance / tail."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("RSA_TC_PP", "0")   # the stamps are implemented in the persistent / one-tile kernels
os.environ["RSA_TC_STAMPS"] = "4"
import bench  # noqa: E402
from paper_2511_19835_b200 import _native as nat  # noqa: E402
from paper_2511_19835_b200.pipeline import _ptr, _stream, workspace_for  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "hv"]
dev = torch.device("cuda", 0)
heads = cfg["heads"]
q, k, v = bench.synth_inputs(torch, cfg, heads, 1234, dev)
shape = nat.make_shape(heads, cfg["t_v"], cfg["t_t"], 128, 128, "bfloat16")
conf = nat.make_config(0.1, 0.0, 0, False, "sparse-rectified")
ws = workspace_for(shape, dev)
out = torch.empty_like(q)
lse = torch.zeros(heads * q.shape[1] + (1 << 16), dtype=torch.float32, device=dev)
lib = nat.lib()
for _ in range(3):
    nat.check(lib.rsa_forward(C.byref(shape), C.byref(conf), _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse),
                              _ptr(ws), _stream()))
torch.cuda.synchronize()
st = lse[:2 * 148 * 2].view(torch.int64).view(148, 2).cpu().numpy().astype(np.float64)
t0 = st[:, 0].min()
end = (st[:, 1] - t0) / 1e3
start = (st[:, 0] - t0) / 1e3
print(f"CTA start spread {start.max():.1f} us; end: min {end.min():.1f} median {np.median(end):.1f} "
      f"max {end.max():.1f} us; tail (max - median) {end.max() - np.median(end):.1f} us "
      f"= {100 * (end.max() - np.median(end)) / end.max():.2f} % of the kernel")
