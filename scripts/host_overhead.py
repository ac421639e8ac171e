"""Host (CPU) cost per ks_matmul call: many calls back to back without
synchronisation on tiny problems (GPU time << host time), wall clock / call."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ksgen, paper_2405_15013_b200 as ksb
from paper_2405_15013_b200 import ks
dev = torch.device("cuda:0")
lib = ks.load_library()
for ps, layout, math in [("2,4,4,2", "bsf", "fp32"), ("1,64,64,1", "bsf", "fp32"), ("1,64,64,1", "bsl", "fp32"),
                         ("1,64,64,1", "bsf", "tf32"), ("1,64,64,1", "bsl", "tf32"), ("1,64,64,4", "bsf", "tf32")]:
    p = tuple(map(int, ps.split(",")))
    f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1))
    if math == "tf32":
        f.set_math(ksb.MATH_TF32)
    B = 256
    X = torch.randn((B, f.N) if layout == "bsf" else (f.N, B), device=dev)
    Y = torch.empty((B, f.M) if layout == "bsf" else (f.M, B), device=dev)
    lay = ks._layout(layout)
    xp, yp = ctypes_x = ks._dev_ptr(X, "X"), ks._dev_ptr(Y, "Y")
    for _ in range(50):
        lib.ks_matmul(f.handle, xp, yp, B, lay, None)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        lib.ks_matmul(f.handle, xp, yp, B, lay, None)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"pattern": p, "layout": layout, "math": math, "plan": f.plan(B, layout),
                      "host_us_per_call": round((t1 - t0) / n * 1e6, 2), "total_us_per_call": round((t2 - t0) / n * 1e6, 2)}))
