#!/usr/bin/env python
"""Hot SASS of an exported ncu source page (`ncu -i rep --page source --csv | gzip`): the instructions that make up
the top share of executed warp instructions of one captured launch, with opcode histogram.
    ncu_source_hot.py <source.csv.gz> [launch index = last] [top N = 40]"""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
want = int(sys.argv[2]) if len(sys.argv) > 2 else -1
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
launches, cur = [], None
with gzip.open(path, "rt") as fh:
    for row in csv.reader(fh):
        if row and row[0] == "Kernel Name":
            cur = {"name": row[1], "rows": [], "hdr": None}
            launches.append(cur)
        elif row and row[0] == "Address":
            cur["hdr"] = row
        elif cur is not None and cur["hdr"] and len(row) >= 6:
            cur["rows"].append(row)
L = launches[want]
h = L["hdr"]
ia, isrc, iex, isamp = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("# Samples")
rows = [(int(r[iex] or 0), int(r[isamp] or 0), r[isrc].strip(), k) for k, r in enumerate(L["rows"])]
tot = sum(r[0] for r in rows)
tots = sum(r[1] for r in rows)
print(f"{L['name']}: {len(rows)} SASS lines, {tot} warp instructions executed, {tots} samples")
hist = collections.Counter()
for ex, sm, src, k in rows:
    hist[src.split()[0].split(".")[0] if not src.startswith("@") else src.split()[1].split(".")[0]] += ex
print("opcode histogram (share of executed):", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in hist.most_common(14)))
# contiguous hot regions: lines executed >= 1/4 of the hottest line
mx = max(r[0] for r in rows)
hot = [r for r in rows if r[0] >= mx / 4]
print(f"lines executed >= max/4: {len(hot)} lines, {100 * sum(r[0] for r in hot) / tot:.1f}% of executed, {100 * sum(r[1] for r in hot) / max(tots, 1):.1f}% of samples")
for ex, sm, src, k in sorted(rows, key=lambda r: -r[0])[:top]:
    print(f"{k:6d} {ex:12d} {100 * ex / tot:5.2f}% samp {sm:6d}  {src[:90]}")

# basic blocks: maximal runs of consecutive lines with the same execution count
blocks, start = [], 0
for k in range(1, len(rows) + 1):
    if k == len(rows) or rows[k][0] != rows[start][0]:
        blocks.append((rows[start][0] * (k - start), rows[start][0], start, k - start, sum(r[1] for r in rows[start:k])))
        start = k
print("\nhottest blocks (runs of lines with equal execution count):")
for totex, ex, s, n, samp in sorted(blocks, key=lambda b: -b[0])[:14]:
    ops = collections.Counter(r[2].split()[0].split(".")[0] if not r[2].startswith("@") else r[2].split()[1].split(".")[0] for r in rows[s:s + n])
    print(f"  lines {s:6d}+{n:4d}  x{ex:11d}  = {100 * totex / tot:5.2f}% of executed, {100 * samp / max(tots, 1):5.2f}% of samples   " +
          " ".join(f"{k}:{v}" for k, v in ops.most_common(8)))
