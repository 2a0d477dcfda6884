"""tcgen05 vs CUDA-core K3 on a small bf16 problem (repeat to catch races):
    python tools/tc_vs_simt.py [t_t] [weight_threshold] [adjacency_radius]"""
import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2511_19835_b200 as rsa
from oracle import rsa_oracle as O
d, block, t_t = 128, 128, int(sys.argv[1]) if len(sys.argv) > 1 else 0
heads = 2
t_v = block * 12
per_head = []
for h in range(heads):
    qv, qt, k, v = O.gen_synthetic(100 + h, t_v, max(t_t, 1), d, block, (1, 1, t_v), 1.0, 2.0, 0.3)
    qt, k, v = qt[:t_t], k[:t_v + t_t], v[:t_v + t_t]
    per_head.append(tuple(O.round_to_bf16(x) for x in (qv, qt, k, v)))
bf = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).cuda()
q = torch.stack([torch.cat([bf(a), bf(b)]) for a, b, _, _ in per_head])
k = torch.stack([bf(x[2]) for x in per_head]); v = torch.stack([bf(x[3]) for x in per_head])
kw = dict(num_text_tokens=t_t, block=block, top_k_fraction=0.2, weight_threshold=float(sys.argv[2]) if len(sys.argv) > 2 else 0.3,
          adjacency_radius=int(sys.argv[3]) if len(sys.argv) > 3 else 1, force_text_blocks=True, check_status=True)
a = rsa.rectified_sparse_attention(q, k, v, kernel="tcgen05", **kw).float()
b = rsa.rectified_sparse_attention(q, k, v, kernel="simt", **kw).float()
diff = (a - b).abs().amax(dim=-1)
bad = torch.nonzero(diff > 1e-2)
print("t_t", t_t, "max diff", diff.max().item(), "bad rows", bad.shape[0], bad[:10].tolist())
