#!/usr/bin/env python3
"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container only (needs /root/reference, numpy, scipy):

    python tests/golden/make_golden.py

1. Copies /root/reference/pkg to a scratch dir and runs the reference's own
   ``scripts/gen_fixtures.py`` there (the shipped tree lacks the RSAT goldens,
   SURVEY.md section 0), then packs every fixture into reference_fixtures.npz.
2. Imports the reference package and records pipeline outputs on seeded
   inputs: tiny fp64/fp32 problems (full outputs), cfg1-shaped bf16-valued
   problems (masks, factors, compensation, a_pool, sampled output rows) and one
   HunyuanVideo-shaped and one Wan-shaped head (pooled path only: masks + R).

Nothing here runs on the GPU box; the fixtures it writes are committed.
"""

import json
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(HERE.parent.parent))

from oracle.rsa_oracle import round_to_bf16  # noqa: E402  (input rounding helper only)


def reference_fixtures(scratch: Path) -> None:
    copy = scratch / "pkg"
    shutil.copytree(REF, copy)
    subprocess.run([sys.executable, "scripts/gen_fixtures.py"], cwd=copy, check=True)
    sys.path.insert(0, str(copy / "src"))
    from rectattn.rsat import read_rsat
    fx = copy / "tests" / "fixtures"
    arrays = {p.stem: read_rsat(p) for p in sorted(fx.glob("*.rsat"))}
    arrays["scalars_json"] = np.frombuffer((fx / "scalars.json").read_bytes(), dtype=np.uint8)
    arrays["demo_sweep_csv"] = np.frombuffer((fx / "demo_sweep.csv").read_bytes(), dtype=np.uint8)
    np.savez_compressed(HERE / "reference_fixtures.npz", **arrays)
    print("reference fixtures:", sorted(arrays))


def run_ref(rt, q_video, q_text, k, v, block, f, p, r, force, variant):
    prob = rt.AttentionProblem(q_video=q_video, q_text=q_text, k=k, v=v,
                               d=q_video.shape[1], block=block)
    cfg = rt.SparsityConfig(top_k_fraction=f, weight_threshold=p,
                            adjacency_radius=r, force_text_blocks=force)
    return rt.rectified_attention_pipeline(prob, cfg, variant=variant)


TINY_CASES = [
    # (seed, t_v, t_t, d, block, dtype, f, p, r, force)
    (0, 32, 6, 8, 4, "f8", 0.25, 0.3, 1, True),
    (1, 32, 7, 8, 4, "f8", 0.2, 0.4, 1, False),
    (2, 64, 10, 8, 8, "f8", 0.25, 0.3, 1, True),
    (3, 16, 0, 8, 4, "f8", 0.5, 0.0, 0, False),
    (4, 64, 9, 16, 8, "f4", 1.0, 0.0, 0, False),
    (5, 64, 8, 16, 8, "f4", 0.3, 0.5, 0, False),
    (6, 48, 5, 16, 16, "f4", 0.4, 0.2, 2, True),
    (7, 24, 3, 8, 1, "f8", 0.3, 0.3, 1, True),
    (8, 96, 13, 32, 8, "f4", 0.1, 0.0, 0, False),
    (9, 128, 32, 32, 16, "f4", 0.2, 0.6, 1, False),
]


def tiny_goldens(rt) -> None:
    out = {}
    for i, (seed, t_v, t_t, d, block, dt, f, p, r, force) in enumerate(TINY_CASES):
        rng = np.random.default_rng(seed)
        dtype = np.dtype(dt)
        qv = rng.standard_normal((t_v, d)).astype(dtype)
        qt = rng.standard_normal((t_t, d)).astype(dtype)
        k = rng.standard_normal((t_v + t_t, d)).astype(dtype)
        v = rng.standard_normal((t_v + t_t, d)).astype(dtype)
        out[f"c{i}_meta"] = np.array([seed, t_v, t_t, d, block, int(dt == "f8"),
                                      f, p, r, int(force)], dtype=np.float64)
        for name, arr in (("qv", qv), ("qt", qt), ("k", k), ("v", v)):
            out[f"c{i}_{name}"] = arr
        for variant in rt.VARIANTS:
            res = run_ref(rt, qv, qt, k, v, block, f, p, r, force, variant)
            tag = f"c{i}_{variant}"
            out[f"{tag}_o_video"] = res.output.o_video
            out[f"{tag}_o_text"] = res.output.o_text
            out[f"{tag}_lse"] = res.output.row_log_denominators
            if variant == "sparse-rectified":
                out[f"c{i}_mask"] = res.sparse_mask.mask
                out[f"c{i}_importance"] = res.sparse_mask.importance
                out[f"c{i}_comp"] = res.comp_mask.mask
                out[f"c{i}_r"] = res.factors.r
                out[f"c{i}_a_pool"] = res.implicit.a_pool
                out[f"c{i}_q_pool"] = res.pooled.q_pool
                out[f"c{i}_v_pool"] = res.pooled.v_pool
                out[f"c{i}_k_mix"] = res.pooled.k_mix_pool
    np.savez_compressed(HERE / "tiny_pipeline.npz", **out)
    print("tiny cases:", len(TINY_CASES))


CFG1 = dict(t_v=3840, t_t=256, d=64, block=64, grid=(1, 60, 64))
CFG1_FRACTIONS = (0.5, 0.25, 0.1, 0.05)
CFG1_THRESHOLDS = (0.0, 0.5)
ROW_STRIDE = 32


def cfg1_inputs(rt, seed):
    spec = rt.SyntheticSpec(seed=seed, t_v=CFG1["t_v"], t_t=CFG1["t_t"], d=CFG1["d"],
                            block=CFG1["block"], grid_dims=CFG1["grid"],
                            locality_strength=1.0, text_norm_boost=2.0,
                            intra_block_noise=0.3, precision="single")
    prob = rt.gen_synthetic(spec)
    return tuple(round_to_bf16(getattr(prob, n)) for n in ("q_video", "q_text", "k", "v"))


def cfg1_goldens(rt) -> None:
    out = {}
    for seed in (42, 43):
        qv, qt, k, v = cfg1_inputs(rt, seed)
        out[f"s{seed}_input_checksum"] = np.array(
            [float(np.abs(x).astype(np.float64).sum()) for x in (qv, qt, k, v)])
        for f in CFG1_FRACTIONS:
            for p in CFG1_THRESHOLDS:
                for variant in rt.VARIANTS:
                    if variant == "full" and (f, p) != (CFG1_FRACTIONS[0], 0.0):
                        continue
                    res = run_ref(rt, qv, qt, k, v, CFG1["block"], f, p, 0, False, variant)
                    tag = f"s{seed}_f{f}_p{p}_{variant}"
                    out[f"{tag}_o_rows"] = res.output.o_video[::ROW_STRIDE]
                    out[f"{tag}_ot_rows"] = res.output.o_text[::ROW_STRIDE // 4]
                    if variant == "sparse-rectified":
                        out[f"s{seed}_f{f}_p{p}_mask"] = np.packbits(res.sparse_mask.mask, axis=1)
                        out[f"s{seed}_f{f}_p{p}_r"] = res.factors.r
                out[f"s{seed}_comp"] = np.packbits(res.comp_mask.mask, axis=1)
                out[f"s{seed}_a_pool"] = res.implicit.a_pool
    np.savez_compressed(HERE / "cfg1_pipeline.npz", **out)
    print("cfg1 goldens written")


HV = dict(t_v=118784, t_t=256, d=128, block=128, grid=(29, 64, 64))
WAN = dict(t_v=75520, t_t=0, d=128, block=128)


def pooled_path_golden(rt, qv, qt, k, v, block, f):
    """Reference pooled path only (no kernel): mask and rectification factors."""
    from rectattn.core import partition, pool_problem
    from rectattn.ipar import implicit_full_attention
    from rectattn.masks import build_sparse_mask
    from rectattn.rectify import rectification_factors
    prob = rt.AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=qv.shape[1], block=block)
    grid = partition(prob)
    pooled = pool_problem(prob, grid)
    imp = implicit_full_attention(prob, pooled, grid)
    cfg = rt.SparsityConfig(top_k_fraction=f, weight_threshold=0.0,
                            adjacency_radius=0, force_text_blocks=False)
    sparse = build_sparse_mask(imp.a_pool, cfg, grid)
    r = rectification_factors(imp.a_pool, sparse).r
    # margin audit: gap between the k-th and (k+1)-th pooled weight per row
    srt = -np.sort(-imp.a_pool, axis=1)
    kk = sparse.importance.sum(axis=1)
    gap = (srt[np.arange(len(kk)), kk - 1] - srt[np.arange(len(kk)), np.minimum(kk, srt.shape[1] - 1)])
    rel_gap = gap / srt[np.arange(len(kk)), kk - 1]
    return np.packbits(sparse.mask, axis=1), r, float(rel_gap.min())


def large_goldens(rt) -> None:
    out = {}
    spec = rt.SyntheticSpec(seed=42, t_v=HV["t_v"], t_t=HV["t_t"], d=HV["d"],
                            block=HV["block"], grid_dims=HV["grid"],
                            locality_strength=1.0, text_norm_boost=2.0,
                            intra_block_noise=0.3, precision="single")
    prob = rt.gen_synthetic(spec)
    qv, qt, k, v = (round_to_bf16(getattr(prob, n)) for n in ("q_video", "q_text", "k", "v"))
    for f in (0.1, 0.05):
        mask, r, gap = pooled_path_golden(rt, qv, qt, k, v, HV["block"], f)
        out[f"hv_s42_f{f}_mask"] = mask
        out[f"hv_s42_f{f}_r"] = r
        out[f"hv_s42_f{f}_min_rel_gap"] = np.array([gap])
        print(f"HV f={f}: min relative k-th gap {gap:.3g}")
    rng = np.random.default_rng(42)
    t = WAN["t_v"]
    qv = round_to_bf16(rng.standard_normal((t, WAN["d"])).astype(np.float32))
    k = round_to_bf16(rng.standard_normal((t, WAN["d"])).astype(np.float32))
    v = round_to_bf16(rng.standard_normal((t, WAN["d"])).astype(np.float32))
    qt = np.zeros((0, WAN["d"]), dtype=np.float32)
    mask, r, gap = pooled_path_golden(rt, qv, qt, k, v, WAN["block"], 0.1)
    out["wan_s42_f0.1_mask"] = mask
    out["wan_s42_f0.1_r"] = r
    out["wan_s42_f0.1_min_rel_gap"] = np.array([gap])
    print(f"Wan f=0.1: min relative k-th gap {gap:.3g}")
    np.savez_compressed(HERE / "large_masks.npz", **out)


# Query blocks whose outputs are recorded at the headline shapes (the full
# reference head is run; only these rows are stored, to keep the fixture small).
def headline_query_blocks(n_q: int, count: int = 64) -> np.ndarray:
    rng = np.random.default_rng(2511)
    pick = set(rng.choice(n_q, count - 2, replace=False).tolist()) | {0, n_q - 1}
    return np.array(sorted(pick), dtype=np.int64)


HEADLINE_ROWS = np.arange(0, 128, 16)      # 8 rows of every sampled query block


def headline_goldens(rt) -> None:
    """The whole reference pipeline (sparse-rectified, f=0.1, p=0) on one
    HunyuanVideo head and one Wan head, outputs recorded on sampled rows; and
    HunyuanVideo masks at the cumulative-weight rule p = 0.3 (paper) / 0.5."""
    import time
    out = {}
    spec = rt.SyntheticSpec(seed=42, t_v=HV["t_v"], t_t=HV["t_t"], d=HV["d"],
                            block=HV["block"], grid_dims=HV["grid"],
                            locality_strength=1.0, text_norm_boost=2.0,
                            intra_block_noise=0.3, precision="single")
    prob = rt.gen_synthetic(spec)
    hv = [round_to_bf16(getattr(prob, n)) for n in ("q_video", "q_text", "k", "v")]
    rng = np.random.default_rng(42)
    t = WAN["t_v"]
    wan = [round_to_bf16(rng.standard_normal((t, WAN["d"])).astype(np.float32)) for _ in range(3)]
    wan = [wan[0], np.zeros((0, WAN["d"]), dtype=np.float32), wan[1], wan[2]]
    for tag, (qv, qt, k, v), block in (("hv", hv, HV["block"]), ("wan", wan, WAN["block"])):
        t0 = time.perf_counter()
        res = run_ref(rt, qv, qt, k, v, block, 0.1, 0.0, 0, False, "sparse-rectified")
        dt = time.perf_counter() - t0
        qb = headline_query_blocks(qv.shape[0] // block)
        rows = (qb[:, None] * block + HEADLINE_ROWS[None, :]).ravel()
        lse_rows = (qb[:, None] * block + np.arange(block)[None, :]).ravel()
        out[f"{tag}_query_blocks"] = qb
        out[f"{tag}_rows"] = rows
        out[f"{tag}_o_video_rows"] = res.output.o_video[rows]
        out[f"{tag}_o_text"] = res.output.o_text
        out[f"{tag}_lse_blocks"] = res.output.row_log_denominators[lse_rows]
        out[f"{tag}_mask"] = np.packbits(res.sparse_mask.mask, axis=1)
        out[f"{tag}_seconds"] = np.array([dt])
        print(f"{tag}: reference pipeline {dt:.1f} s")
    for p in (0.3, 0.5):
        prob_hv = rt.AttentionProblem(q_video=hv[0], q_text=hv[1], k=hv[2], v=hv[3],
                                      d=HV["d"], block=HV["block"])
        from rectattn.core import partition, pool_problem
        from rectattn.ipar import implicit_full_attention
        from rectattn.masks import build_sparse_mask
        from rectattn.rectify import rectification_factors
        grid = partition(prob_hv)
        imp = implicit_full_attention(prob_hv, pool_problem(prob_hv, grid), grid)
        cfg = rt.SparsityConfig(top_k_fraction=0.1, weight_threshold=p,
                                adjacency_radius=0, force_text_blocks=False)
        sparse = build_sparse_mask(imp.a_pool, cfg, grid)
        out[f"hv_p{p}_mask"] = np.packbits(sparse.mask, axis=1)
        out[f"hv_p{p}_r"] = rectification_factors(imp.a_pool, sparse).r
        k_floor = int(np.ceil(0.1 * grid.n_kv))
        binds = int((sparse.mask.sum(axis=1) > k_floor).sum())
        out[f"hv_p{p}_rows_binding"] = np.array([binds])
        print(f"HV p={p}: cumulative-weight rule binds on {binds} of {grid.n_q} rows")
    np.savez_compressed(HERE / "headline_outputs.npz", **out)


MORTON_GRIDS = ((2, 4, 4), (3, 5, 7), (1, 60, 64), (29, 4, 6), (5, 16, 12))


def morton_goldens(rt) -> None:
    """rectattn.core.morton_permutation (core.py:276-291) on a few grids, and a
    reorder_morton round trip of a cfg1-style problem (core.py:294-318)."""
    out = {}
    for g in MORTON_GRIDS:
        out["perm_%d_%d_%d" % g] = rt.core.morton_permutation(g).astype(np.int32)
    np.savez_compressed(HERE / "morton_perms.npz", **out)


DIAG_CASES = ((3, 96, 20, 16, 8), (5, 128, 0, 8, 16), (7, 64, 37, 32, 16))


def diag_goldens(rt) -> None:
    """Reference validation diagnostics on small problems (random_problem
    inputs, regenerated from the seed by the tests): gain_error(with_exact=True)
    (masks.py:189-219), denominator_equivalence_report (metrics.py:90-113),
    gapr_condition_agreement (metrics.py:116-124)."""
    from oracle import rsa_oracle as O
    from rectattn.masks import gain_error
    from rectattn.metrics import denominator_equivalence_report, gapr_condition_agreement
    out = {}
    for seed, t_v, t_t, d, b in DIAG_CASES:
        qv, qt, k, v = O.random_problem(seed, t_v=t_v, t_t=t_t, d=d)
        prob = rt.AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=d, block=b)
        grid = rt.partition(prob)
        pooled = rt.pool_problem(prob, grid)
        ge = gain_error(prob, pooled, grid, with_exact=True)
        rep = denominator_equivalence_report(prob, pooled, grid)
        tag = f"s{seed}"
        out[f"{tag}_gain"], out[f"{tag}_error"] = ge.gain, ge.error
        out[f"{tag}_exact_gain"], out[f"{tag}_exact_error"] = ge.exact_gain, ge.exact_error
        out[f"{tag}_s_sum"], out[f"{tag}_s_sum_pool"] = rep.s_sum, rep.s_sum_pool
        out[f"{tag}_satisfied"] = np.array(rep.satisfied_fraction)
        out[f"{tag}_agreement"] = np.array(gapr_condition_agreement(prob, pooled, grid))
    np.savez_compressed(HERE / "diagnostics.npz", **out)


def rsat_goldens(rt) -> None:
    """Bytes of RSAT files written by the reference writer (rsat.py:17-35)."""
    import tempfile as tf
    from rectattn.rsat import write_rsat
    rng = np.random.default_rng(5)
    arrays = {"f32_2d": rng.standard_normal((7, 5)).astype(np.float32),
              "f64_3d": rng.standard_normal((2, 3, 4)), "f32_1d": np.arange(6, dtype=np.float32)}
    out = {}
    with tf.TemporaryDirectory() as tmp:
        for name, a in arrays.items():
            p = Path(tmp) / f"{name}.rsat"
            write_rsat(p, a)
            out[name] = a
            out[name + "_bytes"] = np.frombuffer(p.read_bytes(), dtype=np.uint8)
    np.savez_compressed(HERE / "rsat_files.npz", **out)


HARNESS_CASES = ((21, 128, 20, 16, 16, 0.25), (22, 256, 0, 32, 32, 0.1))


def harness_goldens(rt) -> None:
    """rectattn.harness.run_variants (harness.py:177-220) on small fp64 problems."""
    from oracle import rsa_oracle as O
    from rectattn.harness import run_variants
    out = {}
    for seed, t_v, t_t, d, b, f in HARNESS_CASES:
        qv, qt, k, v = O.random_problem(seed, t_v=t_v, t_t=t_t, d=d)
        prob = rt.AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=d, block=b)
        reps = run_variants(prob, rt.SparsityConfig(f, 0.0, 0, False), rt.VARIANTS)
        for name, r in reps.items():
            tag = f"s{seed}_{name}"
            out[tag] = np.array([r.normalized_l1, r.cosine_similarity, r.sparsity, r.flops_full,
                                 r.flops_sparse, r.flops_overhead,
                                 np.nan if r.gapr_agreement is None else r.gapr_agreement, float(r.checks_passed)])
    np.savez_compressed(HERE / "harness_variants.npz", **out)


def main():
    if "--harness-only" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        import rectattn as rt
        harness_goldens(rt)
        return
    if "--rsat-only" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        import rectattn as rt
        rsat_goldens(rt)
        return
    if "--diag-only" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        import rectattn as rt
        diag_goldens(rt)
        return
    if "--headline-only" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        import rectattn as rt
        headline_goldens(rt)
        return
    if "--morton-only" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        import rectattn as rt
        morton_goldens(rt)
        return
    with tempfile.TemporaryDirectory() as tmp:
        reference_fixtures(Path(tmp))
        import rectattn as rt
        tiny_goldens(rt)
        cfg1_goldens(rt)
        morton_goldens(rt)
        diag_goldens(rt)
        rsat_goldens(rt)
        harness_goldens(rt)
        if "--no-large" not in sys.argv:
            large_goldens(rt)
            headline_goldens(rt)
    (HERE / "README.md").write_text(
        "Golden fixtures generated by `python tests/golden/make_golden.py` from the\n"
        "reference package at /root/reference/pkg (see the script docstring).\n"
        f"numpy {np.__version__}.\n")


if __name__ == "__main__":
    main()
