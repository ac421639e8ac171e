"""Pivot an A/B jsonl (ks_time.py rows) into a table of GB/s per tag."""
import collections
import json
import statistics
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
by = collections.defaultdict(dict)
tags = []
for r in rows:
    by[(r["layout"], tuple(r["pattern"]))][r["tag"]] = r["gbs"]
    if r["tag"] not in tags:
        tags.append(r["tag"])
print(" " * 26 + " ".join(f"{t:>7s}" for t in tags))
for k, v in by.items():
    print(f"{k[0]} {str(k[1]):20s} " + " ".join(f"{v.get(t, 0):7.0f}" for t in tags))
for lay in ("bsf", "bsl"):
    for t in tags:
        vals = [v[t] for k, v in by.items() if k[0] == lay and t in v]
        if vals:
            print(lay, t, "median", round(statistics.median(vals)), "n", len(vals))
