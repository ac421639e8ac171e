"""Warp-stall mix and instruction mix from ncu source-page CSVs (gpurun_out/prof_*.sass.csv.gz).

    python scripts/stall_summary.py [files...]
"""
import csv
import glob
import gzip
import io
import json
import sys


def summarize(path):
    rows = list(csv.reader(io.TextIOWrapper(gzip.open(path), "utf-8")))
    hdr, data = rows[1], rows[2:]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = {hdr[i]: 0 for i in cols}
    mix = {}
    iexec = hdr.index("Instructions Executed")
    for r in data:
        if len(r) < len(hdr):
            continue
        for i in cols:
            try:
                tot[hdr[i]] += int(r[i])
            except (ValueError, IndexError):
                pass
        toks = r[1].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        try:
            mix[op] = mix.get(op, 0) + int(r[iexec])
        except ValueError:
            pass
    s = sum(tot.values()) or 1
    t = sum(mix.values()) or 1
    return {"stalls": {k: round(v / s, 3) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v / s >= 0.01},
            "inst_mix": {k: round(v / t, 3) for k, v in sorted(mix.items(), key=lambda x: -x[1])[:12]}}


if __name__ == "__main__":
    files = sys.argv[1:] or sorted(glob.glob("gpurun_out/prof_*.sass.csv.gz"))
    print(json.dumps({f.split("/")[-1].split(".")[0]: summarize(f) for f in files}, indent=1))
