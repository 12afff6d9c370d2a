"""Per-source-line warp-stall samples of an ncu --set full report (cuda,sass view), top N lines
across all files: python tools/ncu_lines.py REPORT [N]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, agg, tot = "?", [], 0
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) > 6 and r[0] and r[0] != "Line No" and r[0].isdigit():
        s = int(r[4]) if r[4].isdigit() else 0
        tot += s
        agg.append((s, f"{fname}:{r[0]}", r[1][:90], r[7]))
agg.sort(reverse=True)
print(f"total samples {tot}")
for s, loc, src, ninst in agg[:top]:
    print(f"{s / max(tot, 1):6.1%} {loc:18s} inst={ninst:>10s}  {src}")
