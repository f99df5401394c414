"""Registers / spills per kernel entry from csrc/ptxas.log (build_lib.py -v output)."""
import re
import subprocess
import sys

log = sys.argv[1] if len(sys.argv) > 1 else "paper_2401_11324_b200/csrc/ptxas.log"
pat = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
spill = ""
for line in open(log):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if pat in cur:
            print(f"{m.group(1):>4} regs {spill:<16} {cur}")
        cur, spill = None, ""
