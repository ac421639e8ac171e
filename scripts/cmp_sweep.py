"""Compare two sweep JSONs (bench_sweep.py output) per pattern and layout."""
import json
import statistics as st
import sys


def rows(path):
    d = json.load(open(path))
    k = [k for k, v in d.items() if isinstance(v, list)][0]
    return d, {tuple(r["pattern"]): r for r in d[k]}


old, om = rows(sys.argv[1])
new, nm = rows(sys.argv[2])
lay = sys.argv[3] if len(sys.argv) > 3 else "bsf"
hbm = float(sys.argv[4]) if len(sys.argv) > 4 else 6549.0
for k in ["median_speedup_bsf", "median_speedup_bsl", "median_speedup_min_over_layouts", "win_rate_min_over_layouts"]:
    print(k, old.get(k), new.get(k))
g = [r[f"{lay}_ks_gbs"] for r in nm.values()]
print(lay, "median GB/s", st.median(g), "frac", round(st.median(g) / hbm, 3))
for p, r in nm.items():
    o = om.get(p)
    if o is None:
        continue
    print(list(p), r[f"{lay}_plan"], "us", round(o[f"{lay}_ks_ms"] * 1e3, 1), "->", round(r[f"{lay}_ks_ms"] * 1e3, 1),
          "GB/s", r[f"{lay}_ks_gbs"], "spd", r[f"{lay}_speedup"])
