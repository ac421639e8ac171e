"""One TF32 call for the compute-sanitizer synccheck triage: pattern, layout, knobs (or -1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, ksgen, paper_2405_15013_b200 as ksb
p = tuple(int(v) for v in sys.argv[1].split(","))
lay = sys.argv[2]
knobs = int(sys.argv[3]) if len(sys.argv) > 3 else -1
B = 260 if lay == "bsf" else 256
f = ksb.Factor(*p, ksgen.k4_uniform(*p, seed=3)).set_math(ksb.MATH_TF32)
if knobs >= 0:
    f.set_knobs(knobs)
X = torch.randn((B, f.N) if lay == "bsf" else (f.N, B), device="cuda")
ksb.matmul(f, X, layout=lay)
torch.cuda.synchronize()
print("done", p, lay, knobs, f.plan(B, lay))
