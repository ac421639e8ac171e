"""Offline B200 autotune of the launch-plan knobs (PAPER.md:735
"presets", "auto-tuned per pattern ... and per GPU").

For every configs[2] sweep pattern (B = 25088) and every configs[3]/[4] factor
(ViT-S at B = 25088, GPT-2 at B = 65536), per layout and math (FP32, TF32),
time each relevant knob set through ks_set_knobs (L2 flushed, median of R
reps), check the result against the rules' result (FP32 knobs are
bit-identical by design, R11; TF32 within the 5e-3 contract), and keep the
fastest only when it beats the rules by more than `--margin`.  Writes JSON
(profiles/r02/autotune.json); scripts/gen_presets.py turns it into
csrc/ks_presets.inc.

    python scripts/autotune.py --out gpurun_out/autotune.json [--reps 10]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ksgen  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402
from paper_2405_15013_b200 import ks  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", required=True)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--margin", type=float, default=0.03)
ap.add_argument("--limit", type=int, default=0)
ap.add_argument("--only", default="", help="restrict to math:layout pairs, e.g. tf32:bsl")
args = ap.parse_args()

dev = torch.device("cuda:0")
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size, dtype=torch.uint8, device=dev)
work = [(p, ksgen.configs.SWEEP_BATCH) for p in ksgen.grid.sweep_patterns()]
work += [(p, ksgen.configs.VIT_BATCH) for p in ksgen.configs.VIT_UP + ksgen.configs.VIT_DOWN]
work += [(p, ksgen.configs.GPT2_BATCH) for p in dict.fromkeys(ksgen.configs.GPT2_DOWN + ksgen.configs.GPT2_UP)]
if args.limit:
    work = work[: args.limit]


def timeit(fn):
    for _ in range(3):
        fn()
    ts = []
    for r in range(args.reps):
        flush.fill_(r & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def candidates(p, layout, math, rules):
    a, b, c, d = p
    out = {rules}
    if math == "tf32":
        if layout == "bsl" or d == 1:
            out |= {rules | ks.KNOB_TF32_V2, rules | ks.KNOB_TF32_V2 | ks.KNOB_V2_NKB2}
            if layout == "bsl":           # the v1 kernel with / without MN-major A
                out |= {(rules & ~ks.KNOB_TF32_V2) ^ ks.KNOB_TF32_MN, rules & ~ks.KNOB_TF32_V2 & ~ks.KNOB_TF32_MN}
        else:
            opts = [0]
            if 2 <= d <= 8:
                opts = [m | x for m in opts for x in (0, ks.KNOB_DENSIFY)]
            if d > 8 and d % 8 == 0 and b > 64:
                opts = [m | x for m in opts for x in (0, ks.KNOB_J8)]
            if d == 2 and b > 128 and b % 256 == 0:
                opts = [m | x for m in opts for x in (0, ks.KNOB_BN256)]
            base = rules & ~(ks.KNOB_DENSIFY | ks.KNOB_J8 | ks.KNOB_BN256)
            out |= {base | m for m in opts}
    else:
        base = rules & ~(ks.KNOB_KB32 | ks.KNOB_FFMA_WS | ks.KNOB_FFMA_WSG | ks.KNOB_FFMA_WSL)
        opts = [ks.KNOB_FFMA_WS | ks.KNOB_FFMA_WSG | ks.KNOB_KB32, ks.KNOB_FFMA_WS | ks.KNOB_FFMA_WSG, 0]
        if layout == "bsf" and d > 1:
            opts.append(ks.KNOB_FFMA_WS | ks.KNOB_KB32)
        if layout == "bsf" and d % 4 == 0:      # the lane-j FFMA2 kernel instead of the four-j one
            opts.append(ks.KNOB_FFMA_WS | ks.KNOB_FFMA_WSG | ks.KNOB_KB32 | ks.KNOB_FFMA_WSL)
        out |= {base | m for m in opts}
    return sorted(out)


rows = []
for p, B in work:
    a, b, c, d = p
    M, N = a * b * d, a * c * d
    K4 = ksgen.k4_uniform(*p, seed=1000)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    Xb = torch.randn((B, N), generator=g, device=dev)
    for math in ("fp32", "tf32"):
        f = ksb.Factor(*p, K4)
        if math == "tf32":
            if b < 16 or c < 16:
                continue
            f.set_math(ksb.MATH_TF32)
        for layout in ("bsf", "bsl"):
            if args.only and f"{math}:{layout}" not in args.only.split(","):
                continue
            X = Xb if layout == "bsf" else Xb.t().contiguous()
            Y = torch.empty((B, M) if layout == "bsf" else (M, B), device=dev)
            f.set_knobs(-1)
            rules, src = f.plan_knobs(B, layout)
            f.plan(B, layout)
            ref = ksb.matmul(f, X, layout=layout).clone()
            res = {}
            for m in candidates(p, layout, math, rules):
                f.set_knobs(m)
                try:
                    plan = f.plan(B, layout)
                    ksb.matmul(f, X, Y, layout=layout)
                    torch.cuda.synchronize()
                except ks.KSError:
                    continue
                if math == "fp32":
                    same = bool(torch.equal(Y, ref))
                else:
                    same = float((Y - ref).abs().max() / ref.abs().max()) <= 5e-3
                if not same:
                    print("MISMATCH", p, layout, math, m, flush=True)
                    continue
                res[m] = (timeit(lambda: ksb.matmul(f, X, Y, layout=layout)), plan)
            f.set_knobs(-1)
            t_rules = res[rules][0]
            best = min(res, key=lambda m: res[m][0])
            keep = best if res[best][0] < (1 - args.margin) * t_rules else rules
            row = {"pattern": list(p), "B": B, "lgB": B.bit_length() - 1, "layout": layout, "math": math,
                   "rules": rules, "best": keep, "us": {str(m): round(t * 1e3, 2) for m, (t, _) in res.items()},
                   "plans": {str(m): pl for m, (_, pl) in res.items()},
                   "speedup_vs_rules": round(t_rules / res[keep][0], 4)}
            rows.append(row)
            print(json.dumps(row), flush=True)
            del X, Y, ref
        f.free()
    del Xb
    torch.cuda.empty_cache()

with open(args.out, "w") as fh:
    json.dump({"device": torch.cuda.get_device_name(dev), "reps": args.reps, "margin": args.margin, "rows": rows}, fh)
print("wrote", args.out, len(rows), "rows")
