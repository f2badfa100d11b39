"""Aggregate ncu warp-stall samples per CUDA source line (from a --import-source capture
compiled with -lineinfo):  python tools/ncu_lines.py REPORT.ncu-rep [launch_index] [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, cur, path = {}, None, ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) < 5 or r[0] == "Line No":
        continue
    if r[0]:
        cur = (path, int(r[0]), r[1].strip()[:90])
    if cur and r[4].isdigit():
        agg[cur] = agg.get(cur, 0) + int(r[4])
tot = sum(agg.values()) or 1
print(f"total samples {tot}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100.0 * v / tot:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
