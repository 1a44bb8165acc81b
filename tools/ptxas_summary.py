"""Registers / spills per kernel instance from the ptxas -v logs of the last build
(paper_1706_10086_b200/build/*.ptxas.txt): python tools/ptxas_summary.py [filter]"""
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
flt = sys.argv[1] if len(sys.argv) > 1 else ""
for f in sorted(glob.glob(os.path.join(ROOT, "paper_1706_10086_b200", "build", "*.ptxas.txt"))):
    cur = None
    spill = None
    for line in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            cur = re.sub(r"\(.*", "", cur).replace("dg::", "")
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            spill = (int(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            if flt in cur:
                print(f"{int(m.group(1)):4d} regs  spill st/ld {spill[0]:4d}/{spill[1]:4d}  {cur}")
            cur = None
