"""Small calls of every hot-path kernel for compute-sanitizer (tools/sanitize.sh):
cfg1 (d = B = 64, the persistent tcgen05 K3), a d = B = 128 problem with
ragged text (the paired-tile K3, ping-pong K3 and persistent K3), and the
fp32 CUDA-core K3 -- each checked against the oracle so a sanitizer run
that changes results fails loudly."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2511_19835_b200 as rsa  # noqa: E402
from oracle import rsa_oracle as O  # noqa: E402


def bf(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).cuda()


def check(got, ref, what):
    err = float(np.abs(got - ref).max())
    cos = O.cosine(got, ref)
    assert err <= 2e-2 and cos >= 0.999, (what, err, cos)
    print(f"{what}: max-abs {err:.2e} cos {cos:.6f}")


# cfg1 shape, bf16, persistent K3 (d = B = 64)
qv, qt, k, v = (O.round_to_bf16(x) for x in O.gen_synthetic(42, 3840, 256, 64, 64, (1, 60, 64), 1.0, 2.0, 0.3))
prob = rsa.AttentionProblem(q_video=bf(qv), q_text=bf(qt), k=bf(k), v=bf(v), d=64, block=64)
res = rsa.rectified_attention_pipeline(prob, rsa.SparsityConfig(0.1, 0.0, 0, False))
ref = O.pipeline(qv, qt, k, v, 64, 0.1, 0.0, 0, False, "sparse-rectified")
check(res.output.o_video.float().cpu().numpy(), ref["o_video"], "cfg1 bf16")

# d = B = 128, 2 heads, ragged text: the three tcgen05 K3 kernels
qv, qt, k, v = (O.round_to_bf16(x) for x in O.gen_synthetic(5, 128 * 20, 200, 128, 128, (1, 40, 64), 1.0, 2.0, 0.3))
q = torch.cat([bf(qv), bf(qt)])[None].expand(2, -1, -1).contiguous()
kk, vv = (bf(x)[None].expand(2, -1, -1).contiguous() for x in (k, v))
ref = O.pipeline(qv, qt, k, v, 128, 0.2, 0.0, 0, False, "sparse-rectified")
want = np.concatenate([ref["o_video"], ref["o_text"]])
for kern in ("tcgen05", "tcgen05-pingpong", "tcgen05-persistent"):
    out = rsa.rectified_sparse_attention(q, kk, vv, num_text_tokens=200, block=128, top_k_fraction=0.2, kernel=kern)
    check(out[1].float().cpu().numpy(), want, f"d=B=128 {kern}")

# fp32 (the reference precision): CUDA-core K3
qv, qt, k, v = O.gen_synthetic(7, 1024, 96, 32, 32, (1, 32, 32), 1.0, 2.0, 0.3)
t = lambda x: torch.from_numpy(x).float().cuda()  # noqa: E731
prob = rsa.AttentionProblem(q_video=t(qv), q_text=t(qt), k=t(k), v=t(v), d=32, block=32)
res = rsa.rectified_attention_pipeline(prob, rsa.SparsityConfig(0.2, 0.3, 1, True))
ref = O.pipeline(qv, qt, k, v, 32, 0.2, 0.3, 1, True, "sparse-rectified")
check(res.output.o_video.cpu().numpy(), ref["o_video"], "fp32 CUDA-core")
torch.cuda.synchronize()
print("sanitize workload ok")
