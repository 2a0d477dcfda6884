"""HV call with and without the fused Morton reorder (rsa_forward vs
rsa_forward_permuted), CUDA events, 10 steps after 3 warm-up."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2511_19835_b200 as rsa  # noqa: E402
from paper_2511_19835_b200 import _native as nat  # noqa: E402
from paper_2511_19835_b200.pipeline import workspace_for  # noqa: E402

cfg = bench.CONFIGS["hv"]
dev = torch.device("cuda", 0)
q, k, v = bench.synth_inputs(torch, cfg, cfg["heads"], 1234, dev)
shape = nat.make_shape(cfg["heads"], cfg["t_v"], cfg["t_t"], 128, 128, "bfloat16")
ws = workspace_for(shape, dev)
for morton in (False, True):
    def call():
        return rsa.rectified_sparse_attention(q[None], k[None], v[None], num_text_tokens=cfg["t_t"], block=128,
                                              top_k_fraction=0.1, workspace=ws, grid_dims=cfg["grid"],
                                              morton=morton)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        call()
    e1.record()
    torch.cuda.synchronize()
    print(f"morton={morton}: {e0.elapsed_time(e1) / 10:.3f} ms/call")
