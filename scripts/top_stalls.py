"""Top stalled SASS instructions (ncu source page CSV, gz) with their main stall reasons."""
import csv
import gzip
import io
import sys

rows = list(csv.reader(io.TextIOWrapper(gzip.open(sys.argv[1]), "utf-8")))
hdr, data = rows[1], [r for r in rows[2:] if len(r) >= 10]
isamp = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[isamp] or 0) for r in data)
top = sorted(range(len(data)), key=lambda k: -int(data[k][isamp] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for k in sorted(top):
    r = data[k]
    reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in cols), reverse=True)[:3]
    print(f"{k:5d} {int(r[isamp]) / tot:6.3f} ex={r[iex]:>9s} {r[1].strip()[:60]:60s} " +
          " ".join(f"{n}:{v}" for v, n in reasons if v))
