"""Per-rank work of the head-sharded multi-GPU call, measured on one GPU.

`bench.py --gpus N` shards the HunyuanVideo call's 24 heads over N ranks with
no collective on the data path, so each rank runs the
same pipeline on 24 / N heads.  This times that per-rank call (K1 -> K2 -> K3
through the C ABI, CUDA events over back-to-back calls) for N = 1, 2, 4, 8 on
one B200 and prints the implied strong-scaling efficiency T(24) / (N T(24/N)):
the part of the scaling curve that per-rank load balance (the K3 tail, fixed
per-call costs) decides, before any interconnect effect.

    python tools/rank_projection.py
"""
import ctypes as C
import json
import statistics
import sys
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
q24, k24, v24 = bench.synth_inputs(torch, cfg, 24, 1234, dev)
res = {}
for n in (1, 2, 4, 8):
    h = 24 // n
    q, k, v = q24[:h].contiguous(), k24[:h].contiguous(), v24[:h].contiguous()
    shape = nat.make_shape(h, cfg["t_v"], cfg["t_t"], cfg["d"], cfg["block"], "bfloat16")
    ws = workspace_for(shape, dev)
    out = torch.empty_like(q)
    st, sp = torch.cuda.current_stream(), _stream()
    call = lambda: nat.check(lib.rsa_forward(C.byref(shape), C.byref(conf), _ptr(q), _ptr(k), _ptr(v),  # noqa: E731
                                             _ptr(out), None, _ptr(ws), sp))
    for _ in range(3):
        call()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for e0, e1 in evs:
        e0.record(st)
        call()
        e1.record(st)
    torch.cuda.synchronize()
    res[n] = statistics.median(e0.elapsed_time(e1) for e0, e1 in evs)
    del q, k, v, ws, out
for n, ms in res.items():
    print(json.dumps({"ranks": n, "heads_per_rank": 24 // n, "ms_per_rank_call": round(ms, 3),
                      "strong_scaling_efficiency": round(res[1] / (n * ms), 3)}))
