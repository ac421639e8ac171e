"""configs[2] sweep: the 88 paper-grid patterns with b = c in {48,64,96,128},
a*d <= 64, B = 25088, FP32.

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


def _time(fn, flush, reps, warm=3):
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
    return statistics.median(ts)


def run_sweep(dev, reps: int = 7, patterns=None, math: str = "fp32", check: bool = True):
    import numpy as np
    import torch

    import ksgen
    import paper_2405_15013_b200 as ksb

    pats = patterns or ksgen.grid.sweep_patterns()
    B = ksgen.configs.SWEEP_BATCH
    torch.backends.cuda.matmul.allow_tf32 = (math == "tf32")
    props = torch.cuda.get_device_properties(dev)
    flush = torch.empty(2 * props.L2_cache_size, dtype=torch.uint8, device=dev)
    nmax = max(p[0] * p[2] * p[3] for p in pats)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    Xfull = torch.randn((B, nmax), generator=g, device=dev, dtype=torch.float32)
    rows = []
    for p in pats:
        a, b, c, d = p
        M, N = a * b * d, a * c * d
        K4 = ksgen.k4_uniform(*p, seed=1000)
        f = ksb.Factor(*p, K4)
        if math == "tf32":
            f.set_math(ksb.MATH_TF32)
        Kb = torch.from_numpy(np.ascontiguousarray(K4.transpose(0, 3, 1, 2).reshape(a * d, b, c))).to(dev)
        rec = {"pattern": list(p)}
        for lay in ("bsf", "bsl"):
            X = Xfull[:, :N].contiguous() if lay == "bsf" else Xfull[:, :N].t().contiguous()
            Y = torch.empty((B, M) if lay == "bsf" else (M, B), device=dev)
            t_ks = _time(lambda: ksb.matmul(f, X, Y, layout=lay), flush, reps)
            bfn = bmm_bsf if lay == "bsf" else bmm_bsl
            t_bmm = _time(lambda: bfn(X, Kb, a, b, c, d), flush, reps)
            if check:
                ref = bfn(X, Kb, a, b, c, d)
                ksb.matmul(f, X, Y, layout=lay)
                torch.cuda.synchronize()
                err = float((Y - ref).abs().max() / ref.abs().max())
                rec[f"{lay}_err_vs_bmm"] = err
            byts = 4 * (B * N + a * b * c * d + B * M)
            rec[f"{lay}_plan"] = f.plan(B, lay)
            rec[f"{lay}_ks_ms"] = round(t_ks, 5)
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


if __name__ == "__main__":
    import json
    import sys
    import torch
    dev = torch.device("cuda:0")
    math = sys.argv[1] if len(sys.argv) > 1 else "fp32"
    out = run_sweep(dev, math=math)
    print(json.dumps(out))
