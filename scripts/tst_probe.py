import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ksgen, paper_2405_15013_b200 as ksb  # noqa
import oracle as O  # noqa
p = tuple(int(v) for v in sys.argv[1].split(","))
B = int(sys.argv[2])
K4 = ksgen.k4_uniform(*p, seed=1)
f = ksb.Factor(*p, K4).set_math(ksb.MATH_TF32)
Xn = ksgen.x_normal(B, f.N, seed=0)
Y = ksb.matmul(f, torch.from_numpy(Xn).cuda())
torch.cuda.synchronize()
rows = np.array([0, 1, B // 2, B - 1])
print("ok", p, B, os.environ.get("KS_TF32_DEBUG"), O.normwise_error(Y.cpu().numpy()[rows], O.matmul(p, K4, Xn, rows=rows)))
