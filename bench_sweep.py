"""configs[2] sweep: the 88 paper-grid patterns with b = c in {48,64,96,128},
a*d <= 64, B = 25088, FP32.  Also math = "tf32";
"f32x3" (the FP32-accurate 3xTF32 tensor-core mode, against the true-FP32
bmm); "bf16" / "f16" (NEXT-3, against torch.bmm in the same half format).

For every pattern and layout, times ks_matmul (one fused launch) against the
paper's bmm+permute baseline (App. A listing; BSL = the
"swap first/last dimensions" form) on the same inputs, with
allow_tf32 = False, L2 flushed before every repetition, median of R reps
(PAPER.md:1224 protocol, reduced).  speedup = t_bmm / t_ks; the median over the
88 patterns is reported per layout and with the paper's min-over-layouts rule
(PAPER.md:574-576).  Used by bench.py --sweep.
"""
from __future__ import annotations

import statistics


def bmm_bsf(X, Kb, a, b, c, d):
    import torch
    B = X.shape[0]
    Xp = X.view(B, a, c, d).transpose(-1, -2).reshape(B, a * d, c).contiguous().transpose(0, 1)
    Yp = torch.bmm(Xp, Kb.transpose(-1, -2))
    return Yp.transpose(0, 1).reshape(B, a, d, b).transpose(-1, -2).reshape(B, a * b * d)


def bmm_bsl(X, Kb, a, b, c, d):
    import torch
    B = X.shape[1]
    Xp = X.view(a, c, d, B).permute(0, 2, 1, 3).reshape(a * d, c, B)
    Yp = torch.bmm(Kb, Xp)
    return Yp.view(a, d, b, B).permute(0, 2, 1, 3).reshape(a * b * d, B)


def _time(fn, flush, reps, warm=3, with_iqr=False):
    """Median (and IQR) of `reps` event-timed calls, L2 flushed before each
    (PAPER.md:1224 reports medians with the IQR)."""
    import torch
    for _ in range(warm):
        fn()
    ts = []
    for r in range(reps):
        flush.fill_(r & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    med = statistics.median(ts)
    if not with_iqr:
        return med
    q = statistics.quantiles(ts, n=4) if len(ts) >= 4 else [med, med, med]
    return med, q[2] - q[0]


def run_sweep(dev, reps: int = 7, patterns=None, math: str = "fp32", check: bool = True):
    import torch

    import ksgen
    import paper_2405_15013_b200 as ksb

    pats = patterns or ksgen.grid.sweep_patterns()
    B = ksgen.configs.SWEEP_BATCH
    torch.backends.cuda.matmul.allow_tf32 = (math == "tf32")   # f32x3 is compared with true-FP32 bmm
    dt = {"bf16": torch.bfloat16, "f16": torch.float16}.get(math, torch.float32)
    esize = 2 if dt != torch.float32 else 4
    props = torch.cuda.get_device_properties(dev)
    flush = torch.empty(2 * props.L2_cache_size, dtype=torch.uint8, device=dev)
    nmax = max(p[0] * p[2] * p[3] for p in pats)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    Xfull = torch.randn((B, nmax), generator=g, device=dev, dtype=torch.float32).to(dt)
    rows = []
    for p in pats:
        a, b, c, d = p
        M, N = a * b * d, a * c * d
        K4 = torch.from_numpy(ksgen.k4_uniform(*p, seed=1000)).to(dt)
        f = ksb.Factor(*p, K4)
        if math in ("tf32", "f32x3"):
            f.set_math(ksb.MATH_TF32 if math == "tf32" else ksb.MATH_F32X3)
        Kb = K4.permute(0, 3, 1, 2).reshape(a * d, b, c).contiguous().to(dev)
        rec = {"pattern": list(p)}
        for lay in ("bsf", "bsl"):
            X = Xfull[:, :N].contiguous() if lay == "bsf" else Xfull[:, :N].t().contiguous()
            Y = torch.empty((B, M) if lay == "bsf" else (M, B), device=dev, dtype=dt)
            t_ks, iqr_ks = _time(lambda: ksb.matmul(f, X, Y, layout=lay), flush, reps, with_iqr=True)
            bfn = bmm_bsf if lay == "bsf" else bmm_bsl
            t_bmm = _time(lambda: bfn(X, Kb, a, b, c, d), flush, reps)
            if check:
                ref = bfn(X, Kb, a, b, c, d)
                ksb.matmul(f, X, Y, layout=lay)
                torch.cuda.synchronize()
                err = float((Y.float() - ref.float()).abs().max() / ref.float().abs().max())
                rec[f"{lay}_err_vs_bmm"] = err
            byts = esize * (B * N + a * b * c * d + B * M)
            rec[f"{lay}_plan"] = f.plan(B, lay)
            rec[f"{lay}_ks_ms"] = round(t_ks, 5)
            rec[f"{lay}_ks_iqr_ms"] = round(iqr_ks, 5)
            rec[f"{lay}_bmm_ms"] = round(t_bmm, 5)
            rec[f"{lay}_speedup"] = round(t_bmm / t_ks, 4)
            rec[f"{lay}_ks_gbs"] = round(byts / t_ks / 1e6, 1)
            rec[f"{lay}_ks_tflops"] = round(2 * B * a * b * c * d / t_ks / 1e9, 2)
            del X, Y
        rec["min_speedup"] = round(min(rec["bsf_bmm_ms"], rec["bsl_bmm_ms"]) /
                                   min(rec["bsf_ks_ms"], rec["bsl_ks_ms"]), 4)
        rows.append(rec)
        f.free()
    torch.backends.cuda.matmul.allow_tf32 = False
    med = lambda k: round(statistics.median(r[k] for r in rows), 4)
    return {"math": math, "patterns": len(rows), "batch": B, "reps": reps,
            "median_speedup_bsf": med("bsf_speedup"), "median_speedup_bsl": med("bsl_speedup"),
            "median_speedup_min_over_layouts": med("min_speedup"),
            "win_rate_min_over_layouts": round(sum(r["min_speedup"] > 1 for r in rows) / len(rows), 4),
            "median_tflops_bsf": med("bsf_ks_tflops"), "median_tflops_bsl": med("bsl_ks_tflops"),
            "max_err_vs_bmm": max(max(r.get("bsf_err_vs_bmm", 0), r.get("bsl_err_vs_bmm", 0)) for r in rows),
            "rows": rows}


def permutation_share(dev, reps: int = 7, patterns=None, math: str = "fp32"):
    """SURVEY §8f NEXT-4 / App. E.3 on B200: the share of
    bmm+permute time spent in the two permutations, (dt - dt~)/dt, where dt~
    times the same batched GEMM on the pre-permuted pattern (ad, b, c, 1) whose
    permutations are identities.  BSF, as Fig. 3."""
    import numpy as np
    import torch

    import ksgen

    pats = patterns or ksgen.grid.sweep_patterns()
    B = ksgen.configs.SWEEP_BATCH
    torch.backends.cuda.matmul.allow_tf32 = (math == "tf32")
    props = torch.cuda.get_device_properties(dev)
    flush = torch.empty(2 * props.L2_cache_size, dtype=torch.uint8, device=dev)
    nmax = max(p[0] * p[2] * p[3] for p in pats)
    X = torch.randn((B, nmax), device=dev)
    rows = []
    for (a, b, c, d) in pats:
        Kb = torch.from_numpy(ksgen.k4_uniform(a, b, c, d, seed=1).transpose(0, 3, 1, 2)
                              .reshape(a * d, b, c).copy()).to(dev)
        Xp = X[:, : a * c * d].contiguous()
        t_full = _time(lambda: bmm_bsf(Xp, Kb, a, b, c, d), flush, reps)
        t_noperm = _time(lambda: bmm_bsf(Xp, Kb, a * d, b, c, 1), flush, reps)
        share = max(0.0, min(1.0, (t_full - t_noperm) / t_full))
        rows.append({"pattern": [a, b, c, d], "h": (b + c) / (b * c), "bmm_ms": round(t_full, 5),
                     "bmm_no_perm_ms": round(t_noperm, 5), "perm_share": round(share, 4)})
    torch.backends.cuda.matmul.allow_tf32 = False
    by_h = {}
    for r in rows:
        by_h.setdefault(round(r["h"], 6), []).append(r["perm_share"])
    return {"math": math, "batch": B, "patterns": len(rows),
            "median_share_by_h": {str(k): round(float(np.median(v)), 4) for k, v in sorted(by_h.items())},
            "max_share": max(r["perm_share"] for r in rows), "rows": rows}


def speedup_regression(sweep):
    """The paper's heuristic fit: log speedup = b0 + b1 log density
    + b2 log h, least squares over the sweep, per layout and min-over-layouts."""
    import numpy as np
    out = {}
    for key in ("bsf_speedup", "bsl_speedup", "min_speedup"):
        A, y = [], []
        for r in sweep["rows"]:
            a, b, c, d = r["pattern"]
            A.append([1.0, np.log(1.0 / (a * d)), np.log((b + c) / (b * c))])
            y.append(np.log(r[key]))
        A, y = np.array(A), np.array(y)
        coef, *_ = np.linalg.lstsq(A, y, rcond=None)
        pred = A @ coef
        r2 = 1 - np.sum((y - pred) ** 2) / max(np.sum((y - y.mean()) ** 2), 1e-30)
        out[key] = {"b0": round(float(coef[0]), 4), "b_log_density": round(float(coef[1]), 4),
                    "b_log_h": round(float(coef[2]), 4), "r2": round(float(r2), 4)}
    out["paper_fp32_a100"] = {"b0": 1.69, "b_log_density": -0.031, "b_log_h": 0.325, "adj_r2": 0.697}
    return out


if __name__ == "__main__":
    import json
    import sys
    import torch
    dev = torch.device("cuda:0")
    mode = sys.argv[1] if len(sys.argv) > 1 else "fp32"
    if mode == "perm":
        out = {"fp32": permutation_share(dev, math="fp32"), "tf32": permutation_share(dev, math="tf32")}
    else:
        out = run_sweep(dev, math=mode)
        out["regression"] = speedup_regression(out)
    print(json.dumps(out))
