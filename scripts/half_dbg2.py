import sys, torch, numpy as np
sys.path.insert(0, '.')
import ksgen, paper_2405_15013_b200 as ksb, oracle as O
p = tuple(int(x) for x in sys.argv[1:5])
B = int(sys.argv[5]) if len(sys.argv) > 5 else 264
M, N, _ = O.dims(p)
K4 = torch.from_numpy(ksgen.k4_uniform(*p, seed=1)).to(torch.bfloat16)
X = torch.from_numpy(ksgen.x_normal(B, N, seed=0)).to(torch.bfloat16)
f = ksb.Factor(*p, K4)
print(p, f.plan(B, "bsf"), flush=True)
Y = ksb.matmul(f, X.cuda(), layout="bsf")
torch.cuda.synchronize()
ref = O.matmul(p, K4.float().numpy(), X.float().numpy())
print("err", O.normwise_error(Y.float().cpu().numpy(), ref), flush=True)
