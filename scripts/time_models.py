"""A/B timing of the TF32 model chains (configs[3]/[4]) with mixed-layout
intermediates on / off, per-factor mixed calls, and dense cuBLAS TF32 on the
same shapes.  L2 flushed before every rep; median (IQR) of --reps CUDA-event
times.  Prints one JSON row per measurement."""
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
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--tag", default="")
ap.add_argument("--only", default="")
args = ap.parse_args()
dev = torch.device("cuda:0")
flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size, dtype=torch.uint8, device=dev)
MODELS = {"vit_up": ([(1, 768, 192, 2), (6, 64, 64, 1)], 25088), "vit_down": ([(1, 128, 128, 3), (6, 64, 256, 1)], 25088),
          "gpt2_down": ([(1, 64, 256, 16), (64, 64, 64, 1)], 65536), "gpt2_up": ([(64, 64, 64, 1), (1, 256, 64, 16)], 65536)}


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
    q = statistics.quantiles(ts, n=4)
    return statistics.median(ts), q[2] - q[0]


torch.backends.cuda.matmul.allow_tf32 = True
ksb.set_chain_fusion(False)
for name, (pats, B) in MODELS.items():
    if args.only and name not in args.only.split(","):
        continue
    fs = [ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1000 + l)).set_math(ksb.MATH_TF32) for l, p in enumerate(pats)]
    N, M = fs[-1].N, fs[0].M
    X = torch.randn(B, N, device=dev)
    Y = torch.empty(B, M, device=dev)
    row = {"tag": args.tag, "model": name, "B": B}
    for mixed in (True, False):
        ksb.set_chain_mixed_layouts(mixed)
        row["layouts_" + ("mixed" if mixed else "uniform")] = ksb.chain_layouts(fs, B)[1]
        row["ms_" + ("mixed" if mixed else "uniform")] = timeit(lambda: ksb.chain(fs, X, Y))
    ksb.set_chain_mixed_layouts(True)
    # per factor, in the mixed plan's layouts
    lay = ksb.chain_layouts(fs, B)[1]
    bufs = {}
    src = X
    for t in range(len(fs) - 1, -1, -1):
        f = fs[t]
        yl = lay[t]
        out = torch.empty((B, f.M) if yl == "bsf" else (f.M, B), device=dev)
        xl = lay[t + 1]
        ms = timeit(lambda: ksb.matmul_io(f, src, xl, out, yl))
        byts = 4 * (B * f.N + f.nnz + B * f.M) if hasattr(f, "nnz") else 4 * (B * f.N + B * f.M)
        row[f"factor{t}_{xl}_{yl}"] = {"pattern": list(pats[t]), "ms": ms, "gbs": round(byts / ms[0] / 1e6, 1)}
        src = out
    W = torch.randn(M, N, device=dev)
    row["ms_dense"] = timeit(lambda: torch.matmul(X, W.t(), out=Y))
    byts = 4 * B * (N + M) + 4 * sum(B * f.M for f in fs[1:]) * 2
    row["chain_bytes"] = byts
    row["gbs_mixed"] = round(byts / row["ms_mixed"][0] / 1e6, 1)
    row["speedup_vs_dense_mixed"] = round(row["ms_dense"][0] / row["ms_mixed"][0], 3)
    row["speedup_vs_dense_uniform"] = round(row["ms_dense"][0] / row["ms_uniform"][0], 3)
    print(json.dumps(row), flush=True)
