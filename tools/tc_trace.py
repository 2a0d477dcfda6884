"""Per-step clock trace of one CTA of the tcgen05 kernel (RSA_TC_STAMPS=2)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("RSA_TC_PP", "0")   # the stamps are implemented in the persistent / one-tile kernels
os.environ["RSA_TC_STAMPS"] = "2"
import bench  # noqa: E402
from paper_2511_19835_b200 import _native as nat  # noqa: E402
from paper_2511_19835_b200.pipeline import _ptr, _stream, workspace_for  # noqa: E402

cfg = bench.CONFIGS["hv"]
dev = torch.device("cuda", 0)
heads = 8
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
tiles = heads * (2 * 8 + 928)   # text chunks (2 tiles x 8 chunks) + video tiles per head
tr = lse.view(torch.int64)[tiles * 8: tiles * 8 + 64 * 8].view(64, 8).cpu().numpy().astype(np.int64)
t0 = tr[0, 6]
if os.environ.get("RSA_TC_KERNEL", "2") == "2":
    names = ["mma:K_i ready", "mma:P_i ready", "mma:PV issued", "sm:S_i ready", "sm:S_i loaded", "sm:P_i done",
             "ld:K_i slot", "ld:V_i slot"]
else:
    names = ["mma:K_j ready", "mma:P_j ready", "mma:V_j ready", "sm:S_j ready", "sm:max exch", "sm:P_j done",
             "ld:K_j slot", "ld:V_j slot"]
print("step " + " ".join(f"{n:>14s}" for n in names))
for j in range(0, 40):
    print(f"{j:4d} " + " ".join(f"{(x - t0) if x else -1:14d}" for x in tr[j]))
d = np.diff(tr[:, 3])[5:40]
print("softmax start-to-start per step: median", np.median(d), "clk")
print("softmax busy (S ready -> P done) median", np.median((tr[:, 5] - tr[:, 3])[5:40]))
print("wait P_j -> next S ready median", np.median((tr[1:, 3] - tr[:-1, 5])[5:40]))
