"""Map SASS offsets to CUDA source lines (nvdisasm --print-line-info output of
one function) and print the line (plus inlined-at chain) for each offset.
Usage: SASS_FILE OFF1 OFF2 ..."""
import re
import sys

cur = []
amap = {}
for line in open(sys.argv[1]):
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', line)
    if m:
        cur = [f"{m.group(1).split('/')[-1]}:{m.group(2)}" + (" (inlined)" if "inlined" in m.group(3) else "")]
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*?);', line)
    if m:
        amap[int(m.group(1), 16)] = (cur[0] if cur else "?", m.group(2).strip())
for o in sys.argv[2:]:
    off = int(o, 16)
    print(o, *amap.get(off, ("?", "?")))
