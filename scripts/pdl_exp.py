"""Whole-chain device time of the configs[1] FFT chain, no per-launch tracing
(PDL experiment: run with KS_PDL=0 / 1)."""
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ksb.set_chain_fusion(False)
for _ in range(3):
    ksb.chain(fs, X, Y)
for trace in (False, True):
    ksb.trace_enable(trace)
    ts = []
    for r in range(50):
        flush.fill_(r)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ksb.chain(fs, X, Y)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ksb.trace_enable(False)
    ts.sort()
    print(f"KS_PDL={os.environ.get('KS_PDL', '1')} trace={trace} chain {ts[len(ts)//2]*1e3:.1f} us")
