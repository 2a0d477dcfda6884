"""Measured fp64 GEMM throughput on this box (the K2 roofline denominator):
torch.matmul float64 (cuBLAS DMMA), square 8192 and K2's own strided-batched shape."""
import json, sys
import torch
def tflops(fn, flop, reps=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return flop / (best * 1e-3) / 1e12
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda"); b = torch.randn(n, n, dtype=torch.float64, device="cuda")
sq = tflops(lambda: a @ b, 2 * n ** 3)
# K2 scores GEMM at HunyuanVideo: 24 x [928 x 128] @ [128 x 1186]
q = torch.randn(24, 928, 128, dtype=torch.float64, device="cuda"); kc = torch.randn(24, 128, 1186, dtype=torch.float64, device="cuda")
k2 = tflops(lambda: torch.bmm(q, kc), 2 * 24 * 928 * 1186 * 128)
out = {"fp64_tflops_square8192": sq, "fp64_tflops_k2_scores_shape": k2, "how": "torch.matmul / bmm float64, best of 10, CUDA events"}
print(json.dumps(out))
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"))
