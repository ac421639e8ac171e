"""Small-shape driver for the compute-sanitizer gate (scripts/sanitize.sh):
one call of every kernel family / plan the library has -- generic, stream,
the FFMA families (warp-specialised TMA ring, four-j, all-j, register-staged),
TF32 tcgen05 (BSL transposers, BSF d = 1, BSF J-gather, densified blocks),
3xTF32, BF16 (BSL swap-AB, BSF J), the fused chain and a CUDA-graph chain, with
bias -- checked against the oracle so a silent corruption also fails.  Run it
with KS_TF32_MAXGRID=2 as well so persistent CTAs wrap their rings."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ksgen  # noqa: E402
import oracle as O  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

dev = torch.device("cuda:0")
bad = []


def run(p, lay, math="fp32", kernel=None, B=260, bias=False, knobs=None, act=None):
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=7)
    X = ksgen.x_normal(B, N, seed=8)
    f = ksb.Factor(*p, K4)
    if math == "tf32":
        f.set_math(ksb.MATH_TF32)
    elif math == "f32x3":
        f.set_math(ksb.MATH_F32X3)
    if kernel is not None:
        f.set_kernel(kernel)
    if knobs is not None:
        f.set_knobs(knobs | f.plan_knobs(B, lay)[0])
    bv = ksgen.x_normal(1, M, seed=9)[0] if bias else None
    Xd = torch.from_numpy(X if lay == "bsf" else ksgen.to_bsl(X)).to(dev)
    Y = ksb.matmul(f, Xd, layout=lay, bias=torch.from_numpy(bv).to(dev) if bias else None, act=act)
    torch.cuda.synchronize()
    Yh = Y.cpu().numpy() if lay == "bsf" else Y.cpu().numpy().T
    ref = O.matmul(p, K4, X) + (bv[None, :] if bias else 0)
    if act == "gelu":
        ref = O.gelu(ref)
    e = O.normwise_error(Yh, ref)
    tol = 5e-3 if math == "tf32" else 1e-5
    plan = f.plan(B, lay)
    print(f"{p} {lay} {math} plan={plan} err={e:.2e}", flush=True)
    if e > tol:
        bad.append((p, lay, math, e))


G = ksb.KERNEL_GENERIC
for lay in ("bsf", "bsl"):
    run((2, 3, 2, 3), lay, kernel=G, bias=True)                 # generic
    run((4, 2, 2, 8), lay, bias=True)                           # stream
    run((1, 128, 128, 1), lay, bias=True)                       # FFMA warp-specialised ring
    run((2, 48, 48, 8), lay)                                    # BSF four-j / BSL ring
    run((1, 64, 48, 2), lay)                                    # BSF all-j (d = 2)
    run((1, 64, 48, 6), lay)                                    # BSF register-staged
    run((1, 96, 64, 5), lay, B=77)                              # ragged
    run((1, 64, 64, 1), lay, "tf32", bias=True)                 # tcgen05 BSF d = 1 / BSL transposers
    run((1, 128, 128, 12), lay, "tf32")                         # J-gather (BSF), BSL d = 12
    run((1, 64, 64, 32), lay, "tf32")                           # J = 8 gather
    run((1, 128, 128, 3), lay, "tf32", bias=True)               # densified (BSF, a = 1, d = 3)
    run((1, 768, 192, 2), lay, "tf32", B=200)                   # BN = 256 (BSF) / densified
    run((1, 64, 64, 4), lay, "f32x3")                           # 3xTF32
# round 2: MN-major TF32 BSL, lane-j FFMA BSF, split-c (small B), GELU epilogues, mixed layouts
from paper_2405_15013_b200 import ks  # noqa: E402
run((2, 48, 48, 4), "bsl", "tf32", knobs=ks.KNOB_TF32_MN, bias=True)
run((2, 64, 64, 8), "bsf", knobs=ks.KNOB_FFMA_WS | ks.KNOB_FFMA_WSG | ks.KNOB_FFMA_WSL, bias=True)
run((2, 64, 64, 2), "bsf", B=24, bias=True)
run((1, 64, 64, 4), "bsf", "tf32", bias=True, act="gelu")
run((6, 64, 64, 1), "bsl", bias=True, act="gelu")
for p, (xl, yl) in [((6, 64, 64, 1), ("bsf", "bsl")), ((1, 64, 256, 16), ("bsl", "bsf")), ((1, 256, 64, 16), ("bsf", "bsl"))]:
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=11)
    X = ksgen.x_normal(256, N, seed=12)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    Y = ksb.matmul_io(f, torch.from_numpy(X if xl == "bsf" else ksgen.to_bsl(X)).to(dev), xl, y_layout=yl)
    torch.cuda.synchronize()
    Yh = Y.cpu().numpy() if yl == "bsf" else Y.cpu().numpy().T
    e = O.normwise_error(Yh, O.matmul(p, K4, X))
    print(f"{p} {xl}->{yl} tf32 err={e:.2e}", flush=True)
    if e > 5e-3:
        bad.append((p, xl, yl, e))
# half precision (kind::f16): BSL swap-AB, BSF d = 1 and J-gather
for p, lay in [((2, 96, 96, 3), "bsl"), ((1, 64, 64, 1), "bsf"), ((2, 48, 48, 8), "bsf")]:
    M, N, _ = O.dims(p)
    K4 = torch.from_numpy(ksgen.k4_uniform(*p, seed=3)).bfloat16()
    X = torch.from_numpy(ksgen.x_normal(260, N, seed=4)).bfloat16()
    f = ksb.Factor(*p, K4)
    Xd = (X if lay == "bsf" else X.t().contiguous()).to(dev)
    Y = ksb.matmul(f, Xd, layout=lay).float().cpu().numpy()
    Yh = Y if lay == "bsf" else Y.T
    e = O.normwise_error(Yh, O.matmul(p, K4.float().numpy(), X.float().numpy()))
    print(f"{p} {lay} bf16 err={e:.2e}", flush=True)
    if e > 2 * 2.0 ** -8:
        bad.append((p, lay, "bf16", e))
# chains: fused (NEXT-1), per-factor with PDL, CUDA graph
pats = ksgen.configs.dyadic_patterns(8)
K4s = [ksgen.k4_uniform(*q, seed=1000 + l) for l, q in enumerate(pats, 1)]
fs = [ksb.Factor(*q, k) for q, k in zip(pats, K4s)]
X = ksgen.x_normal(70, 256, seed=0)
ref = O.chain(pats, K4s, X)
for fuse in (True, False):
    ksb.set_chain_fusion(fuse)
    Y = ksb.chain(fs, torch.from_numpy(X).to(dev))
    torch.cuda.synchronize()
    e = O.normwise_error(Y.cpu().numpy(), ref)
    print(f"dyadic chain fused={fuse} err={e:.2e}", flush=True)
    if e > 1e-5:
        bad.append(("chain", fuse, e))
Xd = torch.from_numpy(X).to(dev)
Yg = torch.empty((70, 256), device=dev)
g = ksb.ChainGraph(fs, Xd, Yg)
g.launch()
torch.cuda.synchronize()
e = O.normwise_error(Yg.cpu().numpy(), ref)
print(f"graph chain err={e:.2e}", flush=True)
g.free()
if e > 1e-5:
    bad.append(("graph", e))
print("BAD", bad)
sys.exit(1 if bad else 0)
