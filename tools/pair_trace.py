"""Timeline of CTA 0 of the paired-tile K3 at the HunyuanVideo shape (tools-only
build with -DRSA_PAIR_TRACE, see tools/build_variants.sh):

    RSA_B200_LIB=tools/ab_so/trace.so python tools/pair_trace.py

Prints per-iteration averages: the MMA thread's wait before each of its four
MMA groups (S0, PV1, S1, PV0), the softmax groups' wait for S and busy time
(S ready -> P released), and the period of one iteration (one kv block of both
tiles)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2511_19835_b200 import _native as nat  # noqa: E402
from paper_2511_19835_b200.pipeline import _ptr, _stream, workspace_for  # noqa: E402

cfg = bench.CONFIGS["hv"]
dev = torch.device("cuda", 0)
heads = 24
kernel = sys.argv[1] if len(sys.argv) > 1 else "tcgen05"   # "tcgen05-pingpong": the two-slot kernel
pp = kernel == "tcgen05-pingpong"
q, k, v = bench.synth_inputs(torch, cfg, heads, 1234, dev)
shape = nat.make_shape(heads, cfg["t_v"], cfg["t_t"], 128, 128, "bfloat16", kernel)
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
tr = np.frombuffer(buf, dtype=np.int64).reshape(4, 16384)
mma = tr[0]
n = (16384 // 3) * 3
req = mma[0:n:3] >> 2
kind = mma[0:n:3] & 3
pw = mma[1:n:3]
go = mma[2:n:3]
ok = req > 0
req, kind, pw, go = req[ok], kind[ok], pw[ok], go[ok]
names = ["S", "PV", "-", "-"] if pp else ["S0", "PV1", "S1", "PV0"]
print(f"MMA groups traced: {len(req)}")
for q4 in range(2 if pp else 4):
    sel = kind == q4
    w = (go - req)[sel]
    line = f"  {names[q4]:4s} wait before issue: median {np.median(w):6.0f} mean {w.mean():6.0f}"
    if q4 & 1:
        wp = (pw - req)[sel]
        line += f"  (of which P wait: median {np.median(wp):6.0f} mean {wp.mean():6.0f})"
    print(line)
s0 = np.nonzero(kind == 0)[0]
per = np.diff(req[s0])
print(f"  {'S-group period (one 64-key half of slot 0)' if pp else 'iteration period (S0 to S0)'}: "
      f"median {np.median(per):.0f}  mean {per.mean():.0f} cycles")
issue = np.diff(np.append(go, go[-1]))  # go -> next req
gi = req[1:] - go[:-1]
print(f"  issue time of a group (go -> next request): median {np.median(gi):.0f}")
prod = tr[3]
m2 = (16384 // 2) * 2
preq = prod[0:m2:2]; pgo = prod[1:m2:2]
okp = preq > 0
preq, pgo = preq[okp], pgo[okp]
k = min(len(pgo), len(go))
lat = go[:k] - pgo[:k]
kvw = (go - np.where(kind % 2 == 1, pw, req))[:k]
waited = kvw > 150
print(f"producer: loads {len(pgo)}; slot wait median {np.median(pgo - preq):.0f};"
      f" issue -> MMA go median {np.median(lat):.0f} (groups that waited for K/V: {waited.mean():.2f},"
      f" their issue -> go median {np.median(lat[waited]) if waited.any() else 0:.0f})")
for t in range(2):
    x = tr[1 + t]
    m = (16384 // 6) * 6
    a, b, c1, c2, c3, c = (x[i:m:6] for i in range(6))
    okk = c > 0
    a, b, c1, c2, c3, c = a[okk], b[okk], c1[okk], c2[okk], c3[okk], c[okk]
    print(f"softmax {t}: blocks {len(a)}; wait for S median {np.median(b - a):.0f};"
          f" S ready -> P released median {np.median(c - b):.0f} [S load {np.median(c1 - b):.0f},"
          f" max {np.median(c2 - c1):.0f}, exp+P store {np.median(c3 - c2):.0f}, st wait+release {np.median(c - c3):.0f}];"
          f" period median {np.median(np.diff(b)):.0f}")
i0 = s0[len(s0) // 2]
t0 = req[i0]
print("excerpt (cycles relative to an S0 request): kind req [P ok] go")
for i in range(i0, min(i0 + 8, len(req))):
    print(f"  {names[kind[i]]:4s} {req[i] - t0:8d} {(pw[i] - t0) if kind[i] % 2 and pw[i] else '':>8} {go[i] - t0:8d}")
for t in range(2):
    x = tr[1 + t]
    b = x[1::6]; c = x[5::6]
    j = np.searchsorted(b, t0)
    print(f"  softmax {t}: " + ", ".join(f"[{b[i] - t0}, {c[i] - t0}]" for i in range(j - 1, min(j + 3, len(b)))))
