"""PCIe probe for the e2e leg: pinned H2D alone, D2H alone, both at once (two
streams), 128 MiB each, and ks_chain_host on configs[1] for comparison."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ksgen  # noqa: E402
from ksgen import configs  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

nbytes = 128 << 20
h_in = torch.empty(nbytes // 4).pin_memory()
h_out = torch.empty(nbytes // 4).pin_memory()
d_in = torch.empty(nbytes // 4, device="cuda")
d_out = torch.empty(nbytes // 4, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


out = {}
out["h2d_gbs"] = nbytes / timed(h2d) / 1e6
out["d2h_gbs"] = nbytes / timed(d2h) / 1e6
t = timed(both)
out["bidir_ms"] = t
out["bidir_each_gbs"] = nbytes / t / 1e6
L, B = configs.FFT_L, configs.FFT_BATCH
pats = configs.dyadic_patterns(L)
fs = [ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1000 + l)) for l, p in enumerate(pats, 1)]
Xh = torch.from_numpy(ksgen.x_normal(B, 2 ** L, seed=0)).pin_memory()
Yh = torch.empty((B, 2 ** L)).pin_memory()
t = timed(lambda: ksb.chain_host(fs, Xh, Yh))
out["chain_host_ms"] = t
out["chain_host_copy_gbs_each_way"] = Xh.numel() * 4 / t / 1e6
print(json.dumps(out))
