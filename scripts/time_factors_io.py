"""Time single factors through ks_matmul_io (any in/out layouts), L2 flushed per
rep, median / IQR of CUDA-event times; --knobs forces launch-plan knobs
(ks_set_knobs, -1 = plan).  A/B tool for kernel experiments (env switches
such as KS_TF32_DEBUG are read by libks)."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ksgen  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", required=True, help="a,b,c,d:B:xl:yl;...")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--knobs", type=int, default=-1)
ap.add_argument("--math", default="tf32")
ap.add_argument("--tag", default="")
args = ap.parse_args()
dev = torch.device("cuda:0")
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size, dtype=torch.uint8, device=dev)
for cs in args.cases.split(";"):
    ps, Bs, xl, yl = cs.split(":")
    p = tuple(int(v) for v in ps.split(","))
    B = int(Bs)
    f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1000))
    if args.math == "tf32":
        f.set_math(ksb.MATH_TF32)
    if args.knobs >= 0:
        f.set_knobs(args.knobs)
    X = torch.randn((B, f.N) if xl == "bsf" else (f.N, B), device=dev)
    Y = torch.empty((B, f.M) if yl == "bsf" else (f.M, B), device=dev)
    for _ in range(3):
        ksb.matmul_io(f, X, xl, Y, yl)
    ts = []
    for r in range(args.reps):
        flush.fill_(r & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ksb.matmul_io(f, X, xl, Y, yl)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    q = statistics.quantiles(ts, n=4) if len(ts) >= 2 else [ts[0]] * 3
    t = statistics.median(ts)
    byts = 4 * (B * f.N + f.nnz + B * f.M)
    print(json.dumps({"tag": args.tag, "pattern": list(p), "B": B, "io": f"{xl}->{yl}", "knobs": args.knobs,
                      "us": round(t * 1e3, 2), "iqr_us": round((q[2] - q[0]) * 1e3, 2),
                      "gbs": round(byts / t / 1e6, 1)}), flush=True)
