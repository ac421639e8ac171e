"""Side-by-side of two ks_time.py outputs (A/B): pattern, us and GB/s each, ratio."""
import json
import statistics
import sys

a = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
b = {tuple(r["pattern"]): r for r in (json.loads(l) for l in open(sys.argv[2]) if l.startswith("{"))}
rat, ga, gb = [], [], []
for r in a:
    s = b.get(tuple(r["pattern"]))
    if not s:
        continue
    rat.append(s["us"] / r["us"])
    ga.append(r["gbs"])
    gb.append(s["gbs"])
    print(f"{str(r['pattern']):20s} {r['us']:8.1f} {r['gbs']:7.0f}   {s['us']:8.1f} {s['gbs']:7.0f}   x{s['us'] / r['us']:.3f}")
print(f"median GB/s A {statistics.median(ga):.0f}  B {statistics.median(gb):.0f}   median speedup A over B {statistics.median(rat):.3f}")
