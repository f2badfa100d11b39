"""Registers / spills / shared memory per kernel from csrc/ptxas.log (the release build's
-Xptxas -v output):  python tools/ptxas_table.py [log]"""
import re
import subprocess
import sys

log = sys.argv[1] if len(sys.argv) > 1 else "paper_2508_11553_b200/csrc/ptxas.log"
rows, cur = [], None
for line in open(log):
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = m.group(1)
        try:
            name = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        except OSError:
            pass
        cur = {"kernel": name.replace("tms::", "").split("(")[0], "spill": "", "regs": "", "smem": ""}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = m.group(1)
        s = re.search(r"(\d+) bytes smem", line)
        cur["smem"] = s.group(1) if s else "0"
print("| kernel | registers | spill st/ld (B) | static smem (B) |")
print("|---|---|---|---|")
for r in rows:
    print(f"| `{r['kernel']}` | {r['regs']} | {r['spill']} | {r['smem']} |")
