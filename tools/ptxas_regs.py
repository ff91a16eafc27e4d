"""Registers / spills per kernel from paper_2312_08656_b200/build/ptxas.log (filter by substring)."""
import re
import subprocess
import sys

log = open("paper_2312_08656_b200/build/ptxas.log").read().splitlines()
pat = sys.argv[1] if len(sys.argv) > 1 else ""
name = None
for i, l in enumerate(log):
    m = re.search(r"Function properties for (\S+)", l)
    if m:
        name = m.group(1)
        spill = log[i + 1].strip() if i + 1 < len(log) else ""
        regs = log[i + 2].strip() if i + 2 < len(log) else ""
        if pat in name:
            dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
            r = re.search(r"Used (\d+) registers", regs)
            sp = re.search(r"(\d+) bytes spill stores", spill)
            print(f"{r.group(1) if r else '?':>4} regs  spill {sp.group(1) if sp else '?':>4}  {dem[:150]}")
