"""Top SASS instructions by sampled warp stalls from an ncu source-page CSV
(--page source --csv --print-source sass, gzip'd), with the instruction's
offset in the function, its top stall reasons and executed count.
Usage: FILE [N]"""
import csv
import gzip
import io
import sys

rows = list(csv.reader(io.StringIO(gzip.open(sys.argv[1], "rt").read())))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ia, isrc, iw, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
base = int(data[0][ia], 16)
tot = sum(float(r[iw] or 0) for r in data) or 1
agg = {}
for r in data:
    for i in sc:
        agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
print("total samples", tot, "| overall:", ", ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in
                                                    sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for r in sorted(data, key=lambda r: -float(r[iw] or 0))[:N]:
    w = float(r[iw] or 0)
    top = sorted(((float(r[i] or 0), hdr[i][6:]) for i in sc if r[i] not in ("", "0")), reverse=True)[:3]
    print(f"{100 * w / tot:5.1f}% +0x{int(r[ia], 16) - base:05x} {r[isrc].strip()[:60]:60s} ex={r[iex]:>8s} | " +
          ", ".join(f"{h}={100 * v / tot:.1f}" for v, h in top))
