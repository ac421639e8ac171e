"""Time ks_matmul alone on a list of patterns (B = 25088 unless --batch), one
layout / math, L2 flushed per rep, median of --reps; prints one JSON row per
pattern.  A/B tool for kernel experiments (env switches are read by libks)."""
import argparse
import json
import statistics
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ksgen  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--math", default="tf32")
ap.add_argument("--layout", default="bsl")
ap.add_argument("--batch", type=int, default=25088)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--filter", default="all", help="all | d1 | dgt1 | list of a,b,c,d;...")
ap.add_argument("--tag", default="")
args = ap.parse_args()
dev = torch.device("cuda:0")
pats = ksgen.grid.sweep_patterns()
if args.filter == "d1":
    pats = [p for p in pats if p[3] == 1]
elif args.filter == "dgt1":
    pats = [p for p in pats if p[3] > 1]
elif args.filter != "all":
    pats = [tuple(int(v) for v in s.split(",")) for s in args.filter.split(";")]
B = args.batch
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size, dtype=torch.uint8, device=dev)
nmax = max(p[0] * p[2] * p[3] for p in pats)
g = torch.Generator(device=dev)
g.manual_seed(0)
Xfull = torch.randn((B, nmax), generator=g, device=dev)
for p in pats:
    a, b, c, d = p
    M, N = a * b * d, a * c * d
    f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1000))
    if args.math != "fp32":
        f.set_math({"tf32": ksb.MATH_TF32, "f32x3": ksb.MATH_F32X3}[args.math])
    X = Xfull[:, :N].contiguous() if args.layout == "bsf" else Xfull[:, :N].t().contiguous()
    Y = torch.empty((B, M) if args.layout == "bsf" else (M, B), device=dev)
    for _ in range(3):
        ksb.matmul(f, X, Y, layout=args.layout)
    ts = []
    for r in range(args.reps):
        flush.fill_(r & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ksb.matmul(f, X, Y, layout=args.layout)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    t = statistics.median(ts)
    q1, q3 = statistics.quantiles(ts, n=4)[0], statistics.quantiles(ts, n=4)[2]
    byts = 4 * (B * N + a * b * c * d + B * M)
    print(json.dumps({"tag": args.tag, "pattern": list(p), "layout": args.layout, "math": args.math,
                      "plan": f.plan(B, args.layout), "us": round(t * 1e3, 2), "iqr_us": round((q3 - q1) * 1e3, 2),
                      "gbs": round(byts / t / 1e6, 1)}), flush=True)
    del X, Y
    f.free()
