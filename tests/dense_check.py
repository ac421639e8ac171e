"""TF32 BSF densified super-block path (ks_tf32.cu launch_dense) against the
oracle, run by tests/test_gpu_tf32_dense.py in a subprocess with
KS_TF32_DENSIFY forced (the library reads it once per process)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ksgen  # noqa: E402
import oracle as O  # noqa: E402
import paper_2405_15013_b200 as ksb  # noqa: E402

worst = 0.0
ok = True
for p, B in [((1, 48, 48, 2), 300), ((2, 16, 24, 3), 260), ((1, 128, 128, 3), 300), ((3, 32, 16, 4), 129),
             ((1, 768, 192, 2), 256), ((2, 64, 48, 5), 200), ((1, 32, 32, 7), 140), ((1, 64, 64, 8), 388),
             ((1, 48, 48, 6), 257)]:
    M, N, _ = O.dims(p)
    K4 = ksgen.k4_uniform(*p, seed=3)
    X = ksgen.x_normal(B, N, seed=4)
    f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
    Y = ksb.matmul(f, torch.from_numpy(X).cuda(), layout="bsf")
    bias = ksgen.x_normal(1, M, seed=5)[0]
    Yb = ksb.matmul(f, torch.from_numpy(X).cuda(), layout="bsf", bias=torch.from_numpy(bias).cuda())
    torch.cuda.synchronize()
    Yh, Ybh = Y.cpu().numpy(), Yb.cpu().numpy()
    ref = O.matmul(p, K4, X)
    e = O.normwise_error(Yh, ref)
    # against the oracle on the operands the tensor core sees (K RNA, X truncated)
    Ytf = O.matmul(p, O.round_tf32_rna(K4), O.truncate_tf32(X))
    Yabs = O.matmul(p, np.abs(O.round_tf32_rna(K4)), np.abs(O.truncate_tf32(X)))
    env_ok = bool(np.all(np.abs(Yh - Ytf) <= O.envelope_delta(p[2] * p[3], 0.0) * Yabs + 1e-30))
    bias_ok = np.array_equal(Ybh, (Yh + bias[None, :]).astype(np.float32))
    # small-integer data: exact in TF32 -> bit-exact
    Ki, Xi = ksgen.k4_int(*p, seed=2001), ksgen.x_int(B, N, seed=2000)
    fi = ksb.Factor(*p, Ki).set_math(ksb.MATH_TF32)
    Yi = ksb.matmul(fi, torch.from_numpy(Xi).cuda(), layout="bsf").cpu().numpy()
    int_ok = np.array_equal(Yi.astype(np.float64), O.matmul(p, Ki, Xi))
    print(p, B, "err", e, "env", env_ok, "bias", bias_ok, "int", int_ok, flush=True)
    worst = max(worst, e)
    ok = ok and env_ok and bias_ok and int_ok
sys.exit(0 if ok and worst <= 5e-3 else 1)
