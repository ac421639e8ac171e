"""Run ks_matmul on one pattern (for ncu captures and quick timing).

    python scripts/run_pattern.py a b c d [--layout bsf|bsl] [--math fp32|tf32] [--B 25088] [--reps 5] [--dtype f32|bf16|f16]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import ksgen  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("p", type=int, nargs=4)
ap.add_argument("--layout", default="bsf")
ap.add_argument("--math", default="fp32")
ap.add_argument("--kernel", default="auto")
ap.add_argument("--B", type=int, default=25088)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dtype", default="f32", choices=["f32", "bf16", "f16"])
args = ap.parse_args()
a, b, c, d = args.p
M, N = a * b * d, a * c * d
dt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[args.dtype]
f = ksb.Factor(a, b, c, d, torch.from_numpy(ksgen.k4_uniform(a, b, c, d, seed=1)).to(dt))
if args.math in ("tf32", "f32x3"):
    f.set_math(ksb.MATH_TF32 if args.math == "tf32" else ksb.MATH_F32X3)
if args.kernel != "auto":
    f.set_kernel({"generic": 1, "stream": 2, "ffma": 3, "tf32": 4}[args.kernel])
dev = torch.device("cuda:0")
X = torch.randn((args.B, N) if args.layout == "bsf" else (N, args.B), device=dev).to(dt)
Y = torch.empty((args.B, M) if args.layout == "bsf" else (M, args.B), device=dev, dtype=dt)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ksb.matmul(f, X, Y, layout=args.layout)
torch.cuda.synchronize()
s.record()
for _ in range(args.reps):
    ksb.matmul(f, X, Y, layout=args.layout)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / args.reps
byts = X.element_size() * (args.B * N + a * b * c * d + args.B * M)
print(f"{args.p} {args.layout} {args.math} {args.dtype} plan={f.plan(args.B, args.layout)} {ms*1e3:.1f} us "
      f"{byts/ms/1e6:.0f} GB/s {2*args.B*a*b*c*d/ms/1e9:.1f} TFLOP/s")
