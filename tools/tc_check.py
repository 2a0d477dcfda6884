"""Quick tcgen05-vs-CUDA-core K3 check on small shapes (debug helper)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2511_19835_b200 as rsa  # noqa: E402

torch.manual_seed(0)
for d, block, t_v, t_t in [(128, 128, 128 * 4, 0), (64, 64, 64 * 6, 0), (128, 128, 128 * 8, 200),
                           (64, 64, 64 * 7, 100), (128, 64, 64 * 9, 130), (64, 128, 128 * 5, 60)]:
    q = torch.randn(2, t_v + t_t, d, device="cuda").bfloat16()
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    outs = {}
    for kern in ("simt", "tcgen05"):
        t0 = time.time()
        outs[kern] = rsa.rectified_sparse_attention(q, k, v, num_text_tokens=t_t, block=block, top_k_fraction=0.3,
                                                    kernel=kern, check_status=True)
        torch.cuda.synchronize()
        print(f"  {kern}: {time.time() - t0:.3f}s", flush=True)
    diff = (outs["simt"].float() - outs["tcgen05"].float()).abs().max().item()
    print(f"d={d} B={block} T_v={t_v} T_t={t_t}: max|tc - simt| = {diff:.3e}", flush=True)
