"""The reference's accuracy experiment (harness run_variants) at production
shapes on the GPU: one head of the HunyuanVideo and Wan 2.1 calls (bf16,
gen_synthetic-style inputs as in bench.py), every variant scored against the
dense fp64 reference.  Prints one JSON line per (shape, variant)."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2511_19835_b200 as rsa  # noqa: E402

VARIANTS = ("full", "sparse-unrectified", "sparse-rectified", "sparse-rectified-no-gapr", "compensate-all")
for name in ("hv", "wan"):
    cfg = bench.CONFIGS[name]
    q, k, v = bench.synth_inputs(torch, cfg, 1, 1234, torch.device("cuda", 0))
    tv = cfg["t_v"]
    prob = rsa.AttentionProblem(q_video=q[0, :tv], q_text=q[0, tv:], k=k[0], v=v[0], d=cfg["d"], block=cfg["block"])
    for f in (0.1, 0.05):
        t0 = time.perf_counter()
        reps = rsa.run_variants(prob, rsa.SparsityConfig(f, 0.0, 0, False), VARIANTS)
        dt = time.perf_counter() - t0
        for var, r in reps.items():
            print(json.dumps({"shape": name, "top_k_fraction": f, "variant": var, "normalized_l1": r.normalized_l1,
                              "cosine": r.cosine_similarity, "sparsity": r.sparsity,
                              "gapr_agreement": r.gapr_agreement, "checks_passed": r.checks_passed,
                              "run_variants_s": round(dt, 2)}), flush=True)
