"""Run one half-precision KS matmul per subprocess (so a faulting kernel does not
take the others down) and print its normwise error vs the oracle.
Usage: python scripts/half_debug.py [a,b,c,d,layout ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEFAULT = ["2,128,64,2,bsf", "1,48,48,3,bsf", "3,64,64,4,bsf", "1,96,96,6,bsf", "1,64,64,8,bsf",
           "1,48,64,12,bsf", "1,32,48,16,bsf", "2,16,16,24,bsf"]

CHILD = r"""
import sys; sys.path.insert(0, {root!r})
import numpy as np, torch, ksgen, oracle as O, paper_2405_15013_b200 as ksb
a, b, c, d, lay = {spec!r}.split(","); p = tuple(int(v) for v in (a, b, c, d))
M, N, _ = O.dims(p); B = 264
K4 = torch.from_numpy(ksgen.k4_uniform(*p, seed=3)).bfloat16()
X = torch.from_numpy(ksgen.x_normal(B, N, seed=4)).bfloat16()
f = ksb.Factor(*p, K4)
Xd = (X if lay == "bsf" else X.t().contiguous()).cuda()
Y = ksb.matmul(f, Xd, layout=lay); torch.cuda.synchronize()
Y = Y.float().cpu().numpy(); Y = Y if lay == "bsf" else Y.T
ref = O.matmul(p, K4.float().numpy(), X.float().numpy())
print(p, lay, f.plan(B, lay), "err", O.normwise_error(Y, ref))
"""

for spec in (sys.argv[1:] or DEFAULT):
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, spec=spec)], capture_output=True, text=True,
                       timeout=120)
    print(spec, "rc", r.returncode, r.stdout.strip(), r.stderr.strip().splitlines()[-1:] if r.returncode else "")
