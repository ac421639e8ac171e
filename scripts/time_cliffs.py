"""Ragged-BSL / misaligned-view cases: the FFMA scalar instantiation vs the
generic kernel it replaced and vs the aligned vector path (B = 25088)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ksgen  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=10):
    for _ in range(2):
        fn()
    ts = []
    for r in range(reps):
        flush.fill_(r & 0xFF)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return round(statistics.median(ts), 1)


for p in [(1, 128, 128, 12), (2, 48, 48, 8), (6, 64, 64, 1), (1, 96, 96, 4)]:
    N = p[0] * p[2] * p[3]
    f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1))
    for B, lay, off in [(25088, "bsl", 0), (25087, "bsl", 0), (25088, "bsf", 1), (25088, "bsl", 1)]:
        big = torch.randn(N * B + 1, device="cuda")
        X = big[off:off + N * B].view((B, N) if lay == "bsf" else (N, B))
        res = {}
        for name, k in (("auto", ksb.KERNEL_AUTO), ("generic", ksb.KERNEL_GENERIC)):
            f.set_kernel(k)
            res[name] = t(lambda: ksb.matmul(f, X, layout=lay))
        f.set_kernel(ksb.KERNEL_AUTO)
        print(json.dumps({"pattern": p, "B": B, "layout": lay, "x_offset_floats": off, "plan": f.plan(B, lay),
                          "us": res}), flush=True)
        del big, X
