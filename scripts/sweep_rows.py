"""Per-pattern configs[2] sweep rows (bench_sweep.run_sweep) for one math mode -> JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_sweep  # noqa: E402

math = sys.argv[1] if len(sys.argv) > 1 else "tf32"
out = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/sweep_{math}.json"
r = bench_sweep.run_sweep("cuda:0", reps=7, math=math)
json.dump(r, open(out, "w"), indent=0)
print(math, {k: v for k, v in r.items() if k != "rows"})
