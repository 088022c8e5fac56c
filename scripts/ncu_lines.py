"""Per-source-line hot spots from an ncu report (mixed cuda+sass source page): warp-stall samples,
instructions, shared-memory wavefronts vs ideal, top stall reasons.

    python scripts/ncu_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, acc = "?", None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) < len(hdr) or r[2] != "-":
        continue
    col = {h: r[i] for i, h in enumerate(hdr) if i >= 4}
    key = (fname, int(r[0]))
    d = acc.setdefault(key, {"src": r[1][:100], "samples": 0, "inst": 0, "wf": 0, "wf_ideal": 0, "stalls": {}})
    num = lambda v: int(v) if v.isdigit() else 0  # noqa: E731
    d["samples"] += num(col.get("Warp Stall Sampling (All Samples)", "0"))
    d["inst"] += num(col.get("Instructions Executed", "0"))
    d["wf"] += num(col.get("L1 Wavefronts Shared", "0"))
    d["wf_ideal"] += num(col.get("L1 Wavefronts Shared Ideal", "0"))
    for h, v in col.items():
        if h.startswith("stall_") and "Not Issued" not in h and v.isdigit():
            d["stalls"][h[6:]] = d["stalls"].get(h[6:], 0) + int(v)
tot = sum(d["samples"] for d in acc.values()) or 1
tinst = sum(d["inst"] for d in acc.values()) or 1
print(f"total samples {tot}, warp instructions {tinst}")
for (f, ln), d in sorted(acc.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    st = sorted(((v, k) for k, v in d["stalls"].items()), reverse=True)[:4]
    print(f"{100 * d['samples'] / tot:5.1f}% inst {100 * d['inst'] / tinst:5.1f}% wf {d['wf']:>10} ideal {d['wf_ideal']:>10}"
          f"  {f}:{ln} {d['src']}\n        {st}")
