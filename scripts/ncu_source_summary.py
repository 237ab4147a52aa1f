"""Summarise the SASS source page of an ncu capture (ncu -i REP --page source --csv --print-source sass):
warp instructions executed grouped by execution count (a code region runs once per window, trial or
batch), and the top stall sites.

Usage: python scripts/ncu_source_summary.py SRC.csv [occurrences]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1], newline="")))
occ = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
hi = next(i for i, r in enumerate(rows) if "Source" in r and any("Instructions Executed" == c for c in r))
hdr = rows[hi]
col = {c: i for i, c in enumerate(hdr)}
src_i = col["Source"]
ex_i = col["Instructions Executed"]
st_i = next((col[c] for c in hdr if c.startswith("Warp Stall Sampling (All")), None)


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


ins = []
for r in rows[hi + 1:]:
    if len(r) <= max(src_i, ex_i):
        continue
    ins.append((r[src_i].strip(), num(r[ex_i]), num(r[st_i]) if st_i is not None else 0.0))
total = sum(e for _, e, _ in ins)
stall = sum(s for _, _, s in ins) or 1.0
print(f"# warp instructions executed: {total:.0f}" + (f" = {32 * total / occ:.1f} per 32 occurrences" if occ else ""))
groups = defaultdict(lambda: [0, 0.0])
for _, e, _ in ins:
    if e > 0:
        groups[e][0] += 1
        groups[e][1] += e
print(f"{'exec count':>12s} {'#instr':>7s} {'warp-instr':>14s} {'share':>6s}")
for e, (n, w) in sorted(groups.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{e:12.0f} {n:7d} {w:14.0f} {100 * w / total:5.1f}%")
print("\n# top stall sites (share of stall samples, execution count, SASS)")
for s_, e, st in sorted(ins, key=lambda x: -x[2])[:15]:
    print(f"{100 * st / stall:5.1f}%  n={e:12.0f}  {s_}")
