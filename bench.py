#!/usr/bin/env python3
"""Benchmark of the Rectified SpaAttn hot path on B200 (driver contract).

    python bench.py [--gpus N --steps K --warmup W] [--config hv|wan|cfg1] [--impl ours|reference]

One step = one call of the whole hot path (K1 pool -> K2 select -> K3 block-
sparse attention with the fused IPAR/GAPR epilogue) on the HunyuanVideo 720p
attention shape (BASELINE.json configs[1]): H=24, T_v=118,784 (928 blocks of
128; 118,800 rounded down to the reference's T_v mod B == 0 rule), T_t=256,
d=128, B=128, top_k_fraction 0.1 (90% sparsity), p=0, r=0, no forced text,
variant sparse-rectified.  Inputs are synthetic bf16 (gen_synthetic-style:
per-block Gaussian base + 0.3 noise + 3-D positional embedding for video Q/K,
2x text keys), resident in HBM; they are 2.2 GB, far larger than the 126 MB
L2, so no flush is needed between steps.

Multi-GPU (torchrun, one rank per GPU): the call's heads are sharded across
ranks (strong scaling of one fixed call, no collective on the data path);
ms/call is the max over ranks of the device time.

``--impl reference`` times the reference's own CPU implementation -- the
unmodified rectattn package installed into baseline/_ref (pip --target; it
travels to the GPU box with the repo), through its public
rectified_attention_pipeline -- on the host cores: one COMPLETE head per step
(every query block), the call = heads x the median head (heads are identical
independent problems), in the pinned BLAS environment, plus one
head in the as-shipped environment.  The GPU arm's `cpu_baseline` is the same
measurement on one head.  Without baseline/_ref the oracle port is timed
instead (kind "port").
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (heads, t_video, t_text, d, block, grid_dims)
    "hv": dict(heads=24, t_v=118784, t_t=256, d=128, block=128, grid=(29, 64, 64),
               label="HunyuanVideo 720p x 129f attention (T_v 118,800 -> 118,784)"),
    "wan": dict(heads=40, t_v=75520, t_t=0, d=128, block=128, grid=(59, 32, 40),
                label="Wan 2.1 14B 720p x 81f self-attention (T_v 75,600 -> 75,520)"),
    # the exact HunyuanVideo token count: 928 full blocks + a ragged 16-token block
    # (ragged_video extension; the reference raises BlockSizeError here)
    "hv_exact": dict(heads=24, t_v=118800, t_t=256, d=128, block=128, grid=(33, 45, 80), ragged=True,
                     label="HunyuanVideo 720p x 129f attention, exact T_v 118,800 (ragged final video block)"),
    "cfg1": dict(heads=2, t_v=3840, t_t=256, d=64, block=64, grid=(1, 60, 64),
                 label="synthetic B=1 H=2 N=4096 d=64 block=64 (reference CPU case)"),
}
METRIC = "sparse-attn ms/call + effective TFLOPS @ HunyuanVideo 720p shape, 90% sparsity"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="hv")
    ap.add_argument("--sparsity", type=float, default=0.9)
    ap.add_argument("--weight-threshold", type=float, default=0.0,
                    help="cumulative-weight rule p (masks.py:99-103); the headline config uses 0")
    ap.add_argument("--variant", default="sparse-rectified")
    ap.add_argument("--kernel", default="auto",
                    choices=["auto", "tcgen05", "simt", "tcgen05-pingpong", "tcgen05-persistent"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=1, help="heads per pipelined chunk of the e2e call")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-heads", type=int, default=1, help="complete heads timed by the cpu_baseline leg")
    ap.add_argument("--cpu-warmup", type=int, default=0)
    ap.add_argument("--cpu-worker", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-as-shipped", action="store_true",
                    help="reference arm: skip the one-head timing in the as-shipped BLAS environment")
    ap.add_argument("--as-shipped-timeout", type=float, default=150.0)
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the sparsity sweep / Wan / dense legs appended to the N=1 line")
    ap.add_argument("--heads-per-group", type=int, default=1,
                    help="--input-layout seq: heads per overlapped all-to-all group")
    ap.add_argument("--profile", action="store_true", help="fewer steps, no side legs (for ncu)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo: plumbing check of the multi-rank path (ranks may share one GPU)")
    ap.add_argument("--input-layout", choices=["heads", "seq"], default="heads",
                    help="heads: inputs head-sharded (no collective); seq: video tokens sequence-"
                         "sharded, Ulysses NCCL all-to-all before/after the pipeline (N>1)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers

def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16": d["bf16_tflops"],
                "bf16_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:  # NVML at 20 ms when available (nvidia-smi is too slow for sub-second regions)
            import pynvml as nv
            nv.nvmlInit()
            hd = nv.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}
            mx = nv.nvmlDeviceGetMaxClockInfo(hd, nv.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(hd, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(hd)
                self.rows.append([str(self.index), str(sm), str(mx), "", ""] +
                                 ["Active" if r & bits[k] else "Not Active" for k in
                                  ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")])
                self._stop.wait(0.02)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def synth_inputs(torch, cfg, heads, seed, device):
    """gen_synthetic-style tensors (harness.py:92-126 semantics, torch RNG)."""
    g = torch.Generator(device=device).manual_seed(seed)
    t_v, t_t, d, B = cfg["t_v"], cfg["t_t"], cfg["d"], cfg["block"]
    T = t_v + t_t
    nb = -(-t_v // B)   # (a ragged final block keeps a partial run of its block mean)
    # 3-D sinusoidal positional embedding of the (t, h, w) grid (harness.py:69-89)
    t_, h_, w_ = cfg["grid"]
    d_hw = d // 3
    d_t = d - 2 * d_hw

    def sincos(coord, dim):
        half = dim // 2
        freqs = torch.exp(-math.log(10000.0) * (2 * torch.arange(half + dim % 2, device=device) / max(dim, 1)))
        ang = coord[:, None].double() * freqs[None, :].double()
        out = torch.zeros(coord.shape[0], dim, dtype=torch.float64, device=device)
        out[:, 0::2] = torch.sin(ang)
        out[:, 1::2] = torch.cos(ang[:, :half])
        return out

    idx = torch.arange(t_v, device=device)
    tt, yy, xx = idx // (h_ * w_), (idx // w_) % h_, idx % w_
    pos = torch.cat([sincos(tt, d_t), sincos(yy, d_hw), sincos(xx, d_hw)], dim=1).float()
    q = torch.empty(heads, T, d, dtype=torch.bfloat16, device=device)
    k = torch.empty_like(q)
    v = torch.empty_like(q)
    for h in range(heads):
        qb = torch.randn(nb, d, generator=g, device=device).repeat_interleave(B, 0)[:t_v]
        kb = torch.randn(nb, d, generator=g, device=device).repeat_interleave(B, 0)[:t_v]
        q[h, :t_v] = (qb + 0.3 * torch.randn(t_v, d, generator=g, device=device) + pos).bfloat16()
        k[h, :t_v] = (kb + 0.3 * torch.randn(t_v, d, generator=g, device=device) + pos).bfloat16()
        if t_t:
            q[h, t_v:] = torch.randn(t_t, d, generator=g, device=device).bfloat16()
            k[h, t_v:] = (2.0 * torch.randn(t_t, d, generator=g, device=device)).bfloat16()
        v[h] = torch.randn(T, d, generator=g, device=device).bfloat16()
    return q, k, v


# ----------------------------------------------------------------------------- CPU legs
#
# The reference is a numpy package (rectattn); it is installed, unmodified,
# into baseline/_ref by `pip install --target baseline/_ref` and
# travels to the GPU box with the repo.  Its public entry point
# rectattn.rectified_attention_pipeline is timed on COMPLETE heads (every query
# block, the text queries, the pooled path and the rectification) in a worker
# subprocess, so the BLAS threading environment is set before numpy loads:
#   pinned     OPENBLAS_NUM_THREADS=1, RECTATTN_THREADS=<all cores> (one BLAS
#              thread inside each of the reference's per-query-block threads)
#   as shipped the environment as found (OpenBLAS's own thread pool inside each
#              reference thread -- kernel.py:32-40 default)
# A call is heads x one head's time: heads are identical independent problems
# (SPEC.md:112); only the head count is extrapolated, never query blocks.
# Without baseline/_ref the oracle port (oracle/rsa_oracle.py, bit-identical on
# the goldens) is timed the same way and the line says kind "port".

REF_DIR = ROOT / "baseline" / "_ref"


def _bf16_round(np, x):
    """Round-to-nearest-even fp32 -> bf16 values (the GPU arm's inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def cpu_worker(args):
    """(subprocess) time `--cpu-heads` complete heads after `--cpu-warmup`."""
    import numpy as np
    cfg = CONFIGS[args.config]
    f = 1.0 - args.sparsity
    t_v, t_t, d, B = cfg["t_v"], cfg["t_t"], cfg["d"], cfg["block"]
    kind = "reference" if (REF_DIR / "rectattn").is_dir() and not cfg.get("ragged") else "port"
    if kind == "reference":
        sys.path.insert(0, str(REF_DIR))
        import rectattn as rt
    else:
        from oracle import rsa_oracle as O
    distinct = max(1, min(4, cfg["heads"]))
    cache = {}

    def head(seed):
        if seed in cache:
            return cache[seed]
        if t_t:
            if kind == "reference":
                p = rt.gen_synthetic(rt.SyntheticSpec(seed=seed, t_v=t_v, t_t=t_t, d=d, block=B,
                                                      grid_dims=cfg["grid"], locality_strength=1.0,
                                                      text_norm_boost=2.0, intra_block_noise=0.3,
                                                      precision="single"))
                arrs = (p.q_video, p.q_text, p.k, p.v)
            else:
                tf = (t_v // B) * B
                arrs = O.gen_synthetic(seed, tf, t_t, d, B, (1, tf // B, B) if tf != t_v else cfg["grid"],
                                       1.0, 2.0, 0.3)
                if tf != t_v:   # ragged final video block: N(0,1) rows appended
                    rng = np.random.default_rng(seed)
                    ex = [rng.standard_normal((t_v - tf, d)).astype(np.float32) for _ in range(3)]
                    qv, qt, k, v = arrs
                    arrs = (np.concatenate([qv, ex[0]]), qt, np.concatenate([k[:tf], ex[1], k[tf:]]),
                            np.concatenate([v[:tf], ex[2], v[tf:]]))
        else:   # Wan: T_t = 0, which gen_synthetic rejects -> N(0,1) rows
            rng = np.random.default_rng(seed)
            qv, k, v = (rng.standard_normal((t_v, d)).astype(np.float32) for _ in range(3))
            arrs = (qv, np.zeros((0, d), np.float32), k, v)
        cache[seed] = tuple(_bf16_round(np, x) for x in arrs)
        return cache[seed]

    times = []
    for i in range(args.cpu_warmup + args.cpu_heads):
        qv, qt, k, v = head(42 + i % distinct)
        t0 = time.perf_counter()
        if kind == "reference":
            prob = rt.AttentionProblem(q_video=qv, q_text=qt, k=k, v=v, d=d, block=B)
            conf = rt.SparsityConfig(top_k_fraction=f, weight_threshold=args.weight_threshold,
                                     adjacency_radius=0, force_text_blocks=False)
            rt.rectified_attention_pipeline(prob, conf, variant=args.variant)
        else:
            O.pipeline(qv, qt, k, v, B, f, args.weight_threshold, 0, False, args.variant,
                       ragged=cfg.get("ragged", False))
        dt = time.perf_counter() - t0
        if i >= args.cpu_warmup:
            times.append(dt)
    print(json.dumps({"kind": kind, "head_s": times, "cores": os.cpu_count() or 1,
                      "distinct_heads": distinct}), flush=True)


def cpu_heads(args, heads: int, warmup: int, pinned: bool = True, timeout: float | None = None):
    """Run cpu_worker in a subprocess with the pinned or as-shipped BLAS env."""
    env = dict(os.environ)
    cores = os.cpu_count() or 1
    if pinned:
        env.update(OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1",
                   RECTATTN_THREADS=str(cores))
    else:
        for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "RECTATTN_THREADS"):
            env.pop(k, None)
    cmd = [sys.executable, str(Path(__file__).resolve()), "--cpu-worker", "--config", args.config,
           "--sparsity", str(args.sparsity), "--weight-threshold", str(args.weight_threshold),
           "--variant", args.variant, "--cpu-heads", str(heads), "--cpu-warmup", str(warmup)]
    try:
        res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout, cwd=str(ROOT))
    except subprocess.TimeoutExpired:
        return {"timed_out_s": timeout}
    if res.returncode != 0:
        raise RuntimeError(f"cpu worker failed: {res.stderr[-2000:]}")
    out = json.loads(res.stdout.strip().splitlines()[-1])
    out["env"] = ("OPENBLAS_NUM_THREADS=1, RECTATTN_THREADS=%d" % cores) if pinned else "as shipped (default env)"
    return out


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_dict(cfg, f, args, world, ulysses=False) -> dict:
    """The configuration both arms report (identical keys and values)."""
    return {"workload": cfg["label"], "heads": cfg["heads"], "t_video": cfg["t_v"], "t_text": cfg["t_t"],
            "head_dim": cfg["d"], "block": cfg["block"], "top_k_fraction": round(f, 6),
            "weight_threshold": args.weight_threshold, "adjacency_radius": 0, "force_text_blocks": False,
            "variant": args.variant,
            "parallelism": (f"Ulysses seq->head all-to-all x{world} ({args.dist_backend})" if ulysses
                            else f"head-sharded x{world}"),
            "l2": "inputs 2.2 GB >> 126 MB L2 (no flush needed)" if args.config != "cfg1"
            else "inputs 6 MB; L2 resident"}


def cpu_sample_text(res, heads) -> str:
    n = len(res["head_s"])
    return (f"{n} complete heads (every query block, text queries, pooled path, rectification; "
            f"{res['distinct_heads']} distinct seeds) of {heads}, median per head x {heads} heads")


# ----------------------------------------------------------------------------- main legs

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    f = 1.0 - args.sparsity
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    res = cpu_heads(args, args.steps, args.warmup)
    per_head = statistics.median(res["head_s"])
    ms = per_head * cfg["heads"] * 1e3
    cpu = {"value": ms, "unit": "ms/call", "cores": res["cores"], "kind": res["kind"],
           "sample": cpu_sample_text(res, cfg["heads"]), "env": res["env"], "cpu_model": cpu_model(),
           "per_head_s": per_head, "head_s": res["head_s"]}
    if not args.no_as_shipped:
        shipped = cpu_heads(args, 1, 0, pinned=False, timeout=args.as_shipped_timeout)
        cpu["as_shipped"] = ({"timed_out_after_s": shipped["timed_out_s"]} if "timed_out_s" in shipped else
                             {"per_head_s": shipped["head_s"][0], "ms_per_call": shipped["head_s"][0] *
                              cfg["heads"] * 1e3, "env": shipped["env"], "sample": "1 complete head"})
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms/call", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference gen_synthetic, "
        "bf16-rounded)", "config": config_dict(cfg, f, args, world, args.input_layout == "seq" and world > 1),
        "cpu_baseline": cpu,
        "e2e": {"value": ms, "unit": "ms/call", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _measure(torch, nat, lib, shape, conf, q, k, v, out, ws, steps, warm):
    """Median per-stage event times of `steps` calls (K1, K2, K3) and the whole call."""
    import ctypes as C_
    from paper_2511_19835_b200.pipeline import _ptr, _stream
    st, sp = torch.cuda.current_stream(), _stream()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(warm + steps)]
    # back-to-back calls, one synchronisation: the host enqueues ahead of the
    # GPU, so no event pair brackets host-side launch latency
    for ev in evs:
        ev[0].record(st)
        nat.check(lib.rsa_pool(C_.byref(shape), _ptr(q), _ptr(k), _ptr(v), _ptr(ws), sp))
        ev[1].record(st)
        nat.check(lib.rsa_select(C_.byref(shape), C_.byref(conf), _ptr(ws), sp))
        ev[2].record(st)
        nat.check(lib.rsa_attention(C_.byref(shape), C_.byref(conf), _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                    None, _ptr(ws), sp))
        ev[3].record(st)
    torch.cuda.synchronize()
    rows = [[ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
             ev[0].elapsed_time(ev[3])] for ev in evs[warm:]]
    nat.check(lib.rsa_check_device_status(_ptr(ws), sp))
    med = [statistics.median(r[j] for r in rows) for j in range(4)]
    return {"pool": med[0], "select": med[1], "attention": med[2], "call": med[3]}


def _exec_flops(torch, nat, ws, shape, grid, heads, d, T, t_t, block, dev):
    """Executed FLOPs (metrics.py:85 convention + text rows) and realized sparsity."""
    L = nat.layout(shape)
    bits = ws[L["mask_bits"]:L["mask_bits"] + heads * grid.n_q * grid.n_kv].view(heads, grid.n_q, grid.n_kv)
    mask = (bits & 1).to(torch.int64)
    lens = torch.full((grid.n_kv,), block, dtype=torch.int64, device=dev)
    if grid.n_text_blocks:
        lens[-1] = grid.last_text_block_len
    lens[grid.n_q - 1] = grid.last_video_block_len
    qlens = torch.full((grid.n_q,), block, dtype=torch.int64, device=dev)
    qlens[-1] = grid.last_video_block_len
    pairs = int((mask * lens[None, None, :] * qlens[None, :, None]).sum().item())
    flops = 4 * d * pairs + 4 * t_t * T * d * heads
    return flops, 1.0 - float(mask.sum().item()) / (heads * grid.n_q * grid.n_kv)


def extras(torch, nat, lib, workspace_for, args, q, k, v, out, ws, dev, peak_burst):
    """BASELINE.json configs[2]-[3] on the same run: the sparsity sweep at the
    HunyuanVideo shape (IPAR+GAPR on = sparse-rectified, off = sparse-
    unrectified, and our own dense kernel = the `full` variant) and the Wan 2.1
    shape at 90 %; 5 timed calls after 2 warm-ups each."""
    hv = CONFIGS["hv"]
    heads, T, d = q.shape[0], q.shape[1], q.shape[2]
    shape = nat.make_shape(heads, hv["t_v"], hv["t_t"], d, hv["block"], "bfloat16", args.kernel)
    grid = nat.plan(shape)
    res = {"sweep": [], "note": "ms/call (CUDA events, median of 5 after 2 warm-up); frac = K3 executed "
                                "TFLOP/s / measured burst bf16 peak"}
    for f in (0.5, 0.25, 0.1, 0.05):
        for variant in ("sparse-rectified", "sparse-unrectified"):
            conf = nat.make_config(f, 0.0, 0, False, variant)
            t = _measure(torch, nat, lib, shape, conf, q, k, v, out, ws, 5, 2)
            fl, sp = _exec_flops(torch, nat, ws, shape, grid, heads, d, T, hv["t_t"], hv["block"], dev)
            res["sweep"].append({"top_k_fraction": f, "variant": variant, "ms": t["call"], "kernels_ms": t,
                                 "realized_sparsity": sp, "k3_tflops": fl / (t["attention"] * 1e-3) / 1e12,
                                 "k3_frac": fl / (t["attention"] * 1e-3) / 1e12 / peak_burst})
    conf = nat.make_config(1.0, 0.0, 0, False, "full")
    t = _measure(torch, nat, lib, shape, conf, q, k, v, out, ws, 3, 1)
    fl = 4 * T * T * d * heads
    res["dense_full"] = {"ms": t["call"], "kernels_ms": t, "k3_tflops": fl / (t["attention"] * 1e-3) / 1e12,
                         "k3_frac": fl / (t["attention"] * 1e-3) / 1e12 / peak_burst}
    wan = CONFIGS["wan"]
    qw, kw_, vw = synth_inputs(torch, wan, wan["heads"], 4321, dev)
    ow = torch.empty_like(qw)
    shape_w = nat.make_shape(wan["heads"], wan["t_v"], wan["t_t"], wan["d"], wan["block"], "bfloat16", args.kernel)
    grid_w = nat.plan(shape_w)
    ws_w = workspace_for(shape_w, dev)
    conf = nat.make_config(0.1, 0.0, 0, False, "sparse-rectified")
    t = _measure(torch, nat, lib, shape_w, conf, qw, kw_, vw, ow, ws_w, 5, 2)
    fl, sp = _exec_flops(torch, nat, ws_w, shape_w, grid_w, wan["heads"], wan["d"], wan["t_v"], 0, wan["block"], dev)
    res["wan"] = {"workload": wan["label"], "heads": wan["heads"], "t_video": wan["t_v"], "top_k_fraction": 0.1,
                  "ms": t["call"], "kernels_ms": t, "realized_sparsity": sp,
                  "k3_tflops": fl / (t["attention"] * 1e-3) / 1e12,
                  "k3_frac": fl / (t["attention"] * 1e-3) / 1e12 / peak_burst}
    del qw, kw_, vw, ow, ws_w
    return res


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2511_19835_b200 as rsa
    from paper_2511_19835_b200 import _native as nat
    from paper_2511_19835_b200.pipeline import _ptr, _stream, workspace_for

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())   # --dist-backend gloo smoke runs share one GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    cfg = CONFIGS[args.config]
    f = 1.0 - args.sparsity
    # head sharding: rank r owns heads [lo, hi)
    per = [cfg["heads"] // world + (1 if r < cfg["heads"] % world else 0) for r in range(world)]
    lo = sum(per[:rank])
    heads = per[rank]
    q, k, v = synth_inputs(torch, cfg, heads, 1234 + lo, dev)
    T, d = q.shape[1], q.shape[2]
    shape = nat.make_shape(heads, cfg["t_v"], cfg["t_t"], d, cfg["block"], "bfloat16", args.kernel,
                           ragged_video=cfg.get("ragged", False))
    conf = nat.make_config(f, args.weight_threshold, 0, False, args.variant)
    grid = nat.plan(shape, conf)
    ws = workspace_for(shape, dev)
    out = torch.empty_like(q)
    lib = nat.lib()
    st = torch.cuda.current_stream()
    sptr = _stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def step(record=False):
        if record:
            ev[0].record(st)
        nat.check(lib.rsa_pool(C.byref(shape), _ptr(q), _ptr(k), _ptr(v), _ptr(ws), sptr))
        if record:
            ev[1].record(st)
        nat.check(lib.rsa_select(C.byref(shape), C.byref(conf), _ptr(ws), sptr))
        if record:
            ev[2].record(st)
        nat.check(lib.rsa_attention(C.byref(shape), C.byref(conf), _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                    None, _ptr(ws), sptr))
        if record:
            ev[3].record(st)

    ulysses = args.input_layout == "seq" and world > 1
    if ulysses:
        # every rank holds its T_v/P slice of all heads' video tokens + replicated text
        from paper_2511_19835_b200.parallel import ulysses_attention
        qa, ka, va = synth_inputs(torch, cfg, cfg["heads"], 1234, dev)
        t_v = cfg["t_v"]
        s_loc = t_v // world
        sl = slice(rank * s_loc, (rank + 1) * s_loc)
        uq, uk, uv = (x[None, :, sl].contiguous() for x in (qa, ka, va))
        tq, tk, tv = (x[None, :, t_v:].contiguous() for x in (qa, ka, va))
        del qa, ka, va

        groups = -(-(cfg["heads"] // world) // max(1, args.heads_per_group))
        ukw = dict(block=cfg["block"], top_k_fraction=f, weight_threshold=args.weight_threshold,
                   variant=args.variant, kernel=args.kernel, workspace=ws, check_status=False)

        def step(record=False):
            if record:
                ev[0].record(st)
                ev[1].record(st)
                ev[2].record(st)
            ulysses_attention(uq, uk, uv, tq, tk, tv, heads_per_group=args.heads_per_group, **ukw)
            if record:
                ev[3].record(st)

    for _ in range(args.warmup):
        c0 = nat.last_launch_count()
        step()
        # (a Ulysses step is `groups` rsa_forward calls; the counter holds the last one)
        launches_per_step = nat.last_launch_count() * groups if ulysses else nat.last_launch_count() - c0
    nat.check(lib.rsa_check_device_status(_ptr(ws), sptr))
    torch.cuda.synchronize()

    # executed FLOPs of this rank (metrics.py:85 convention + text rows)
    L = nat.layout(shape)
    bits = ws[L["mask_bits"]:L["mask_bits"] + heads * grid.n_q * grid.n_kv].view(heads, grid.n_q, grid.n_kv)
    mask = (bits & 1).to(torch.int64)
    lens = torch.full((grid.n_kv,), cfg["block"], dtype=torch.int64, device=dev)
    if grid.n_text_blocks:
        lens[-1] = grid.last_text_block_len
    lens[grid.n_q - 1] = grid.last_video_block_len           # (a ragged final video block)
    qlens = torch.full((grid.n_q,), cfg["block"], dtype=torch.int64, device=dev)
    qlens[-1] = grid.last_video_block_len
    # sum over query blocks of (query rows x retained kv tokens)
    retained_pairs = int((mask * lens[None, None, :] * qlens[None, :, None]).sum().item())
    flops_video = 4 * d * retained_pairs
    flops_text = 4 * cfg["t_t"] * T * d * heads
    flops_exec = flops_video + flops_text
    flops_dense = 4 * T * T * d * heads
    sparsity = 1.0 - float(mask.sum().item()) / (heads * grid.n_q * grid.n_kv)

    # ---------------- timed region ----------------
    per_stage = {"pool": [], "select": [], "attention": []}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(st)
        for _ in range(args.steps):
            step(record=False)
        t1.record(st)
        torch.cuda.synchronize()
        # per-kernel split, measured on the launching stream over back-to-back
        # steps (one unrecorded step first, so the host enqueues ahead of the GPU
        # and no event pair brackets host-side launch latency), synchronised once
        n_split = max(2, min(args.steps, 5))
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n_split)]
        step(record=False)
        for i in range(n_split):
            ev[:] = evs[i]
            step(record=True)
        torch.cuda.synchronize()
        for e4 in evs:
            per_stage["pool"].append(e4[0].elapsed_time(e4[1]))
            per_stage["select"].append(e4[1].elapsed_time(e4[2]))
            per_stage["attention"].append(e4[2].elapsed_time(e4[3]))
    if world > 1:
        dist.barrier()
    total_ms = t0.elapsed_time(t1)
    ms_step = total_ms / args.steps
    stage = {k2: statistics.median(vv) for k2, vv in per_stage.items()}
    if world > 1:
        tt = torch.tensor([ms_step, stage["attention"], stage["pool"], stage["select"]], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_step, stage["attention"], stage["pool"], stage["select"] = tt.tolist()
        ft = torch.tensor([flops_exec, flops_dense], dtype=torch.float64, device=dev)
        dist.all_reduce(ft)
        flops_exec, flops_dense = ft.tolist()

    # ---------------- end-to-end through the public API (host buffers) ----------------
    e2e = None
    if not args.profile and args.e2e_steps > 0:
        hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
        out_box = []

        def e2e_step():
            # the public call on HOST tensors: H2D of q/k/v, K1 -> K2 -> K3 and the
            # D2H of the output, pipelined over chunks of heads (rsa_forward_host)
            out_box[:] = [rsa.rectified_sparse_attention(hq[None], hk[None], hv[None], num_text_tokens=cfg["t_t"],
                                                         block=cfg["block"], top_k_fraction=f, weight_threshold=args.weight_threshold,
                                                         variant=args.variant, kernel=args.kernel,
                                                         workspace=ws, heads_per_chunk=args.e2e_chunk,
                                                         ragged_video=cfg.get("ragged", False))]

        e2e_step()
        e2e_step()   # second warm-up: the pinned output buffers come from torch's host cache from here on
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(st)
        for _ in range(args.e2e_steps):
            e2e_step()
        a1.record(st)
        torch.cuda.synchronize()
        e2e_ms = a0.elapsed_time(a1) / args.e2e_steps
        if world > 1:
            tt = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = tt.item()
        nbytes = q.numel() * q.element_size()
        e2e = {"value": e2e_ms, "unit": "ms/call", "h2d_bytes_per_step": 3 * nbytes * world,
               "d2h_bytes_per_step": nbytes * world,
               "heads_per_chunk": args.e2e_chunk,
               "path": "rectified_sparse_attention(pinned host q/k/v) -> host output; H2D, K1-K3 and D2H "
                       "pipelined over head chunks (rsa_forward_host)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peaks = measured_peaks()
    attn_ms = stage["attention"]
    per_rank_exec = flops_exec / world
    achieved = per_rank_exec / (attn_ms * 1e-3) / 1e12
    peak = peaks["bf16"]   # burst: K3 is timed on its own (per-stage events), not inside a seconds-long step
    traffic = None
    tp = ROOT / "profiles" / "attn_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(args.config)
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": ms_step, "unit": "ms/call", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (gen_synthetic-style, torch RNG)",
        "config": config_dict(cfg, f, args, world, ulysses),
        "kernel_choice": args.kernel,
        "tflops_effective": flops_exec / (ms_step * 1e-3) / 1e12,
        "tflops_dense_equivalent": flops_dense / (ms_step * 1e-3) / 1e12,
        "realized_sparsity": sparsity,
        "kernels_ms": stage,
        "roofline": {"bound": "tensor", "kernel": "attn_tc_kernel (K3+K4)", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "frac_of_sustained": achieved / peaks["bf16_sustained"], "peak_src": peaks["src"] + " burst",
                     "traffic": traffic,
                     "algorithmic": f"{per_rank_exec / 1e12:.3f} TFLOP executed per launch "
                                    f"(4*B*d*sum(mask*len) + 4*T_t*T*d)"},
        "gpu_launches": launches_per_step * args.steps,
        "e2e": e2e,
    }
    # the other two stages against their own bounds: K1 streams Q/K/V
    # once from HBM; K2 is fp64 GEMM + per-row work (neither HBM- nor tensor-bound)
    t_all = cfg["t_v"] + cfg["t_t"]
    k1_bytes = (cfg["t_v"] + 2 * t_all) * d * 2 * heads
    n_q, n_cols = grid.n_q, grid.n_cols
    k2_flop = (2 * n_q * n_cols * d + 2 * n_q * grid.n_kv * d) * heads
    fp64_peak = None
    fp = ROOT / "profiles" / "fp64_peak.json"
    if fp.exists():
        try:
            fp64_peak = json.loads(fp.read_text()).get("fp64_tflops_square8192")
        except Exception:
            fp64_peak = None
    if stage.get("pool") and stage.get("select"):
        line["stage_rooflines"] = {
            "K1_pool": {"bound": "hbm", "achieved": k1_bytes / (stage["pool"] * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                        "unit": "GB/s", "frac": k1_bytes / (stage["pool"] * 1e-3) / 1e9 / peaks["hbm_gbs"],
                        "algorithmic": f"{k1_bytes / 1e9:.3f} GB read per launch ((T_v + 2T) * d * 2 per head)"},
            "K2_select": {"bound": "fp64 GEMM + per-row", "achieved": k2_flop / (stage["select"] * 1e-3) / 1e12,
                          "peak": fp64_peak, "unit": "fp64 TFLOP/s",
                          "frac": (k2_flop / (stage["select"] * 1e-3) / 1e12 / fp64_peak) if fp64_peak else None,
                          "algorithmic": f"{k2_flop / 1e9:.2f} GFLOP fp64 per launch (scores + compensation GEMMs); "
                                         "peak: measured fp64 GEMM (profiles/fp64_peak.json, tools/fp64_peak.py)"},
        }
    if not args.profile:
        line["clocks"] = clocks.summary()
    if world == 1 and not args.no_extras and not args.profile and args.config == "hv":
        line["extras"] = extras(torch, nat, lib, workspace_for, args, q, k, v, out, ws, dev, peaks["bf16"])
    if world == 1 and not args.no_cpu_baseline and not args.profile:
        res = cpu_heads(args, args.cpu_heads, args.cpu_warmup)
        per_head = statistics.median(res["head_s"])
        line["cpu_baseline"] = {"value": per_head * cfg["heads"] * 1e3, "unit": "ms/call", "cores": res["cores"],
                                "kind": res["kind"], "sample": cpu_sample_text(res, cfg["heads"]),
                                "env": res["env"], "cpu_model": cpu_model(), "per_head_s": per_head}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(args) -> bool:
    """`--gpus N` (N > 1) outside torchrun: re-launch this command as N ranks
    (torch.distributed.run, 127.0.0.1 rendezvous); rank 0 prints the line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.cpu_worker:
        return False
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.run(cmd).returncode)


def main():
    args = parse()
    if args.cpu_worker:
        cpu_worker(args)
        return
    spawn_ranks(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
