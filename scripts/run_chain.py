"""Time ks_chain on the configs[1] FFT chain (fused and per-factor)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ksgen  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 12
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
pats = ksgen.configs.dyadic_patterns(L)
fs = [ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1000 + l)) for l, p in enumerate(pats, 1)]
N = 2 ** L
X = torch.randn(B, N, device="cuda")
Y = torch.empty_like(X)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for fuse in (True, False):
    ksb.set_chain_fusion(fuse)
    for _ in range(3):
        ksb.chain(fs, X, Y)
    ts = []
    for r in range(20):
        flush.fill_(r)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ksb.chain(fs, X, Y)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"L={L} B={B} fused={fuse} radix={os.environ.get('KS_FUSED_RADIX', '8')} {ms*1e3:.1f} us "
          f"hbm_eff={4*2*B*N/ms/1e6:.0f} GB/s")
