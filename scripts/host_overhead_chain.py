"""Host cost per call through the Python binding (ksb.matmul / ksb.chain, the calls
a user makes) and the raw C ABI, tiny problems, no synchronisation between calls."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ksgen, paper_2405_15013_b200 as ksb  # noqa: E402
from paper_2405_15013_b200 import ks  # noqa: E402
dev = torch.device("cuda:0")
lib = ks.load_library()
p = (2, 4, 4, 2)
f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1))
X = torch.randn((8, f.N), device=dev)
Y = torch.empty((8, f.M), device=dev)
def bench(name, fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"call": name, "host_us_per_call": round((t1 - t0) / n * 1e6, 2),
                      "total_us_per_call": round((t2 - t0) / n * 1e6, 2)}), flush=True)
xp, yp = ks._dev_ptr(X, "X"), ks._dev_ptr(Y, "Y")
bench("lib.ks_matmul", lambda: lib.ks_matmul(f.handle, xp, yp, 8, 0, None))
bench("ksb.matmul", lambda: ksb.matmul(f, X, Y))
bench("ksb.chain[1]", lambda: ksb.chain([f], X, Y))
hs = (ks.ctypes.c_void_p * 1)(f.handle) if hasattr(ks, "ctypes") else None
fs12 = [ksb.Factor(*q, ksgen.k4_uniform(*q, seed=1)) for q in ksgen.configs.dyadic_patterns(12)]
X2 = torch.randn((8, 4096), device=dev)
Y2 = torch.empty((8, 4096), device=dev)
ksb.set_chain_fusion(False)
bench("ksb.chain[12 fft] per-factor", lambda: ksb.chain(fs12, X2, Y2), n=500)
ksb.set_chain_fusion(True)
bench("ksb.chain[12 fft] fused", lambda: ksb.chain(fs12, X2, Y2), n=500)
