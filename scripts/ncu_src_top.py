"""Top source lines by warp-stall samples from an ncu --page source --csv export (cuda+sass rows)."""
import csv
import gzip
import sys

path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
op = gzip.open if path.endswith(".gz") else open
with op(path, "rt") as f:
    rows = list(csv.reader(f))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lines = []
for r in rows[hdr_i + 1:]:
    if len(r) < 5 or not r[0]:
        continue  # sass rows have empty line no
    try:
        samples = int(r[4])
    except ValueError:
        continue
    lines.append((samples, r[0], r[1][:110], {hdr[i]: r[i] for i in stall_cols if r[i] not in ("0", "", "-")}))
tot = sum(x[0] for x in lines)
print("total samples", tot, "| stall columns:", len(stall_cols))
for s, ln, src, st in sorted(lines, reverse=True)[:top]:
    top3 = sorted(((int(v), k) for k, v in st.items() if v.isdigit()), reverse=True)[:4]
    print(f"{s:6d} {100*s/tot:5.1f}% L{ln:>5} {src}\n        {top3}")
