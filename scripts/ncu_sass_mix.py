"""Instruction mix (warp-level executed counts by opcode) and top stall instructions from an
`ncu -i REP --page source --csv` SASS export.   python scripts/ncu_sass_mix.py export.csv [top]"""
import collections
import csv
import sys

path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15
rows = list(csv.reader(open(path)))
hdr = rows[1]
ia, isrc, iexe, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
mix, samples, tot = collections.Counter(), collections.Counter(), 0
hot = []
for r in rows[2:]:
    if len(r) <= iexe:
        continue
    op = r[isrc].strip().split()[0] if r[isrc].strip() else "?"
    if op.startswith("@"):
        op = r[isrc].strip().split()[1]
    base = op.split(".")[0]
    n = int(r[iexe] or 0)
    mix[base] += n
    tot += n
    s = int(r[isamp] or 0)
    samples[base] += s
    hot.append((s, r[ia], r[isrc].strip()))
print(f"total warp instructions {tot:.4g}")
for op, n in mix.most_common(top):
    print(f"  {op:10s} {n:14d} {100 * n / tot:5.1f}%  stall samples {samples[op]}")
print("hottest instructions by stall samples:")
for s, a, src in sorted(hot, reverse=True)[:top]:
    print(f"  {s:7d} {a[-5:]} {src}")
