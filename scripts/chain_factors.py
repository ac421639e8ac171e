"""Per-factor device time of the configs[1] FFT chain (library trace events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ksgen  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

pats = ksgen.configs.dyadic_patterns(12)
fs = [ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1000 + l)) for l, p in enumerate(pats, 1)]
B, N = 8192, 4096
X = torch.randn(B, N, device="cuda")
Y = torch.empty_like(X)
ksb.set_chain_fusion(False)
for _ in range(3):
    ksb.chain(fs, X, Y)
torch.cuda.synchronize()
ksb.trace_enable(True)
reps = 20
for _ in range(reps):
    ksb.chain(fs, X, Y)
torch.cuda.synchronize()
ms, fam, byts = ksb.trace_read()
ksb.trace_enable(False)
L = len(pats)
for t in range(L):
    vals = sorted(ms[t::L])
    p = pats[L - 1 - t]
    print(f"factor {p} {vals[len(vals)//2]*1e3:.1f} us  {byts[t]/vals[len(vals)//2]/1e6:.0f} GB/s")
