"""Summarise an ncu --page source CSV (cuda,sass) into per-source-line stall samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
if len(sys.argv) > 3 and sys.argv[3] == "inst":
    pass
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
si = hdr.index("Warp Stall Sampling (All Samples)")
lines = {}
cur = None
for r in rows[hdr_i + 1:]:
    if len(r) <= si:
        continue
    if r[0].isdigit():
        cur = (int(r[0]), r[1][:100])
        try:
            lines[cur] = lines.get(cur, 0) + float(r[si] or 0)
        except ValueError:
            pass
tot = sum(lines.values()) or 1
for (ln, src), v in sorted(lines.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}%  L{ln:<4d} {src.strip()}")


def inst_by_line(rep, top=30):
    """Per-source-line dynamic warp instructions (Instructions Executed)."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hi]
    ii = h.index("Instructions Executed")
    acc = {}
    for r in rows[hi + 1:]:
        if len(r) > ii and r[0].isdigit():
            try:
                acc[(int(r[0]), r[1][:90])] = acc.get((int(r[0]), r[1][:90]), 0) + float(r[ii] or 0)
            except ValueError:
                pass
    tot = sum(acc.values()) or 1
    print(f"total instructions {tot:.0f}")
    for (ln, src), v in sorted(acc.items(), key=lambda x: -x[1])[:top]:
        print(f"{100 * v / tot:5.1f}% {v:10.0f}  L{ln:<4d} {src.strip()}")
