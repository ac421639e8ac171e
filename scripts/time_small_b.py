"""Small-batch latency: the split-c warp-shuffle kernel against the forced FFMA /
generic families on GEMM-like patterns, B in {1, 8, 32, 64}; per-call device
time of 100 calls replayed from one CUDA graph, median of 5."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ksgen  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

for p in [(1, 128, 128, 1), (2, 48, 48, 8), (6, 64, 64, 1), (1, 768, 192, 2), (64, 64, 64, 1), (1, 64, 256, 16)]:
    for B in (1, 8, 32, 64):
        for lay in ("bsf", "bsl"):
            f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1))
            N = p[0] * p[2] * p[3]
            X = torch.randn((B, N) if lay == "bsf" else (N, B), device="cuda")
            res = {}
            for name, kern in (("splitc", ksb.KERNEL_SPLITC), ("ffma", ksb.KERNEL_FFMA),
                               ("generic", ksb.KERNEL_GENERIC)):
                f.set_kernel(kern)
                try:
                    ksb.matmul(f, X, layout=lay)
                except ksb.KSError:
                    continue
                # 100 calls captured into one CUDA graph and replayed: per-call DEVICE time
                # without the host's per-call overhead (~13 us through Python/ctypes) and
                # below the event timer's ~2 us resolution
                Y = torch.empty((B, f.M) if lay == "bsf" else (f.M, B), device="cuda")
                ksb.matmul(f, X, Y, layout=lay)
                torch.cuda.synchronize()
                s0 = torch.cuda.Stream()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s0):
                    for _ in range(100):
                        ksb.matmul(f, X, Y, layout=lay)
                ts = []
                for _ in range(5):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    g.replay()
                    e.record()
                    e.synchronize()
                    ts.append(s.elapsed_time(e) * 1e3 / 100)
                res[name] = round(statistics.median(ts), 2)
            print(json.dumps({"pattern": p, "B": B, "layout": lay, "us": res}), flush=True)
