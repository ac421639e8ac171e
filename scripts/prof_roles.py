"""Per-role wait breakdown of the TF32 J-kernel (KS_TF32_DEBUG=8 instrumentation:
clock64 counters written over Y).  Prints, per case, the mean over CTAs of each
role's waiting cycles as a fraction of its run time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KS_TF32_DEBUG"] = "8"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ksgen  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

dev = torch.device("cuda:0")
for cs in sys.argv[1].split(";"):
    ps, Bs, xl, yl = cs.split(":")
    p = tuple(int(v) for v in ps.split(","))
    B = int(Bs)
    f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=1000))
    f.set_math(ksb.MATH_TF32)
    X = torch.randn((B, f.N) if xl == "bsf" else (f.N, B), device=dev)
    Y = torch.zeros((B, f.M) if yl == "bsf" else (f.M, B), device=dev)
    for _ in range(3):
        ksb.matmul_io(f, X, xl, Y, yl)
    torch.cuda.synchronize()
    raw = Y.flatten()[: 148 * 32].cpu().numpy().view(np.uint64).reshape(148, 16).astype(np.float64)
    names = ["prod_sempty", "prod_empty", "tr_sfull", "tr_empty", "mma_acce", "mma_full", "epi_accf"]
    tot = {"prod": raw[:, 8], "tr": raw[:, 9], "mma": raw[:, 10], "epi": raw[:, 11]}
    out = {"case": cs, "cycles": float(np.mean(raw[:, 10]))}
    for k, n in enumerate(names):
        role = n.split("_")[0]
        out[n] = round(float(np.mean(raw[:, k] / np.maximum(tot[role], 1))), 3)
    print(json.dumps(out), flush=True)
