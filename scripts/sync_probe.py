import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ksgen, paper_2405_15013_b200 as ksb
p = tuple(int(v) for v in sys.argv[1].split(","))
B = int(sys.argv[2])
f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=3)).set_math(ksb.MATH_TF32)
X = torch.randn(p[0] * p[2] * p[3], B, device="cuda")
ksb.matmul(f, X, layout="bsl")
torch.cuda.synchronize()
print("done", p, B)
