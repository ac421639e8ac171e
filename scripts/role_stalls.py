"""Warp-stall samples of a warp-specialised kernel grouped by source-line
ranges (roles).  Usage: SASS_CSV_GZ NVDISASM_FILE 'role:lo-hi,role:lo-hi,...' [file]"""
import csv
import gzip
import io
import re
import sys

rows = list(csv.reader(io.StringIO(gzip.open(sys.argv[1], "rt").read())))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ia, iw = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
fname = sys.argv[4] if len(sys.argv) > 4 else "ks_tf32.cu"
lmap, cur = {}, None
for line in open(sys.argv[2]):
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', line)
    if m and cur:
        lmap[int(m.group(1), 16)] = cur
roles = [(n, int(a), int(b)) for n, rng in (x.split(":") for x in sys.argv[3].split(",")) for a, b in [rng.split("-")]]
agg, lastrole = {}, "other"
tot = 0.0
for r in data:
    off = int(r[ia], 16) - base
    f, ln = lmap.get(off, ("?", 0))
    role = None
    if f == fname:
        for n, a, b in roles:
            if a <= ln <= b:
                role = n
    role = role or lastrole          # inlined helpers (ks_umma.cuh) inherit the enclosing role
    lastrole = role
    w = float(r[iw] or 0)
    tot += w
    d = agg.setdefault(role, {"samples": 0.0, "inst": 0})
    d["samples"] += w
    d["inst"] += int(r[iex] or 0)
    for i in sc:
        v = float(r[i] or 0)
        if v:
            d[hdr[i][6:]] = d.get(hdr[i][6:], 0) + v
for n, d in sorted(agg.items(), key=lambda kv: -kv[1]["samples"]):
    st = sorted(((v, k) for k, v in d.items() if k not in ("samples", "inst")), reverse=True)[:4]
    print(f"{n:12s} {100 * d['samples'] / tot:5.1f}% inst={d['inst']:>9d} | " +
          ", ".join(f"{k}={100 * v / tot:.1f}" for v, k in st))
