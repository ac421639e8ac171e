"""Does the L2 flush method change small-problem timings?  fill = write a 2xL2
buffer (dirty lines left in L2); fill+read = the same write followed by a
read-only pass over a second 2xL2 buffer (L2 left holding clean lines), so the
flush's own write-back does not land inside the timed region."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ksgen, paper_2405_15013_b200 as ksb
dev = torch.device("cuda:0")
L2 = torch.cuda.get_device_properties(dev).L2_cache_size
fl = torch.empty(2 * L2, dtype=torch.uint8, device=dev)
rd = torch.ones(2 * L2 // 4, dtype=torch.float32, device=dev)
acc = torch.empty((), device=dev)
for ps, layout in [("1,48,48,1", "bsl"), ("1,128,128,1", "bsl"), ("1,128,128,4", "bsl"), ("1,64,64,8", "bsl"),
                   ("4,128,128,16", "bsl"), ("1,128,128,4", "bsf"), ("16,128,128,4", "bsf")]:
    p = tuple(map(int, ps.split(",")))
    f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1000)).set_math(ksb.MATH_TF32)
    B = 25088
    X = torch.randn((B, f.N) if layout == "bsf" else (f.N, B), device=dev)
    Y = torch.empty((B, f.M) if layout == "bsf" else (f.M, B), device=dev)
    out = {}
    for mode in ("fill", "fill+read", "none"):
        ts = []
        for r in range(23):
            if mode != "none":
                fl.fill_(r & 0xFF)
            if mode == "fill+read":
                torch.sum(rd, dim=0, out=acc)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); ksb.matmul(f, X, Y, layout=layout); e.record(); e.synchronize()
            ts.append(s.elapsed_time(e))
        out[mode] = round(statistics.median(ts[3:]) * 1e3, 2)
    byts = 4 * (B * f.N + f.nnz + B * f.M)
    print(json.dumps({"pattern": p, "layout": layout, "us": out, "gbs": {k: round(byts / v / 1e3, 1) for k, v in out.items()}}))
