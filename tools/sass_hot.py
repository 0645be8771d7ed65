"""Group an `ncu --page source --print-source sass --csv` dump into straight-line
runs of equal execution count and print the hottest runs (instruction mix)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie, src, smp = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
seen, data = set(), []
for r in rows[2:]:
    if len(r) > ie and r[0].startswith("0x") and r[0] not in seen:   # the csv repeats every row
        seen.add(r[0])
        data.append((int(r[0], 16), r[src].strip(), int(r[ie] or 0), int(r[smp] or 0)))
tot = sum(d[2] for d in data)
print("total warp instructions", tot, "static", len(data))
base = data[0][0]
out, cur = [], None
for a, s, c, sm in data:
    if cur is None or c != cur[2]:
        if cur:
            out.append(cur)
        cur = [a - base, 0, c, 0, 0, collections.Counter()]
    cur[1] += 1
    cur[3] += c
    cur[4] += sm
    op = s.split()[1] if s.startswith("@") else s.split()[0]
    cur[5][op] += 1
out.append(cur)
out.sort(key=lambda x: -x[3])
for o in out[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{o[0]:#07x} n={o[1]:4d} cnt={o[2]:8d} total={o[3]:10d} ({100 * o[3] / tot:4.1f}%) samples={o[4]:5d}",
          o[5].most_common(5))
