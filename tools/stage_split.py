"""Per-stage event split (K1 / K2 / K3) of the HunyuanVideo call at a given
head count next to the whole rsa_forward call and its host-side enqueue time
(back-to-back calls, one synchronisation).

    python tools/stage_split.py [heads ...]
"""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2511_19835_b200 import _native as nat  # noqa: E402
from paper_2511_19835_b200.pipeline import _ptr, _stream, workspace_for  # noqa: E402

cfg = bench.CONFIGS["hv"]
dev = torch.device("cuda", 0)
lib = nat.lib()
conf = nat.make_config(0.1, 0.0, 0, False, "sparse-rectified")
for h in [int(x) for x in sys.argv[1:]] or [24, 3]:
    q, k, v = bench.synth_inputs(torch, cfg, h, 1234, dev)
    shape = nat.make_shape(h, cfg["t_v"], cfg["t_t"], 128, 128, "bfloat16")
    ws = workspace_for(shape, dev)
    out = torch.empty_like(q)
    st, sp = torch.cuda.current_stream(), _stream()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(12)]
    for e in evs:
        e[0].record(st)
        nat.check(lib.rsa_pool(C.byref(shape), _ptr(q), _ptr(k), _ptr(v), _ptr(ws), sp))
        e[1].record(st)
        nat.check(lib.rsa_select(C.byref(shape), C.byref(conf), _ptr(ws), sp))
        e[2].record(st)
        nat.check(lib.rsa_attention(C.byref(shape), C.byref(conf), _ptr(q), _ptr(k), _ptr(v), _ptr(out), None,
                                    _ptr(ws), sp))
        e[3].record(st)
    torch.cuda.synchronize()
    split = [statistics.median(e[i].elapsed_time(e[i + 1]) for e in evs[2:]) for i in range(3)]
    fw = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(12)]
    host = []
    for e0, e1 in fw:
        e0.record(st)
        t0 = time.perf_counter()
        nat.check(lib.rsa_forward(C.byref(shape), C.byref(conf), _ptr(q), _ptr(k), _ptr(v), _ptr(out), None,
                                  _ptr(ws), sp))
        host.append((time.perf_counter() - t0) * 1e3)
        e1.record(st)
    torch.cuda.synchronize()
    whole = statistics.median(e0.elapsed_time(e1) for e0, e1 in fw[2:])
    print(f"heads {h}: K1 {split[0]:.3f}  K2 {split[1]:.3f}  K3 {split[2]:.3f}  sum {sum(split):.3f}  "
          f"rsa_forward {whole:.3f} ms  host enqueue {statistics.median(host):.3f} ms")
    del q, k, v, ws, out
