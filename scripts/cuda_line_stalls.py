"""Top CUDA source lines by sampled warp stalls from an ncu source-page CSV
(--page source --csv --print-source cuda, gzip'd).  Usage: FILE [N]"""
import csv
import gzip
import io
import sys

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
text = gzip.open(path, "rt").read()
# several files concatenated: each block starts with "File Name"
blocks = text.split('"File Name",')
res = []
for blk in blocks[1:]:
    lines = blk.splitlines()
    fname = lines[0].strip('"').split("/")[-1]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    try:
        iw = hdr.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        continue
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    for r in rows[1:]:
        if len(r) <= iw:
            continue
        try:
            w = float(r[iw] or 0)
        except ValueError:
            continue
        if w <= 0:
            continue
        top = sorted(((float(r[i] or 0), hdr[i]) for i in stall_cols if r[i] not in ("", "0")), reverse=True)[:3]
        res.append((w, fname, r[0], r[1].strip()[:90], top))
tot = sum(x[0] for x in res)
for w, f, ln, src, top in sorted(res, reverse=True)[:N]:
    print(f"{100 * w / tot:5.1f}% {f}:{ln} {src}  | " + ", ".join(f"{h[6:]}={v:.0f}" for v, h in top))
