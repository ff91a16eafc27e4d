"""Top SASS instructions by warp-stall samples from an ncu --set full --import-source report.
usage: python tools/ncu_hot.py REPORT.ncu-rep [N] [kernel-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
blocks = out.split('"Kernel Name"')
for b in blocks[1:]:
    lines = b.split("\n")
    kname = lines[0]
    if len(sys.argv) > 3 and sys.argv[3] not in kname:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ia, isrc, ist, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    data = [r for r in rows[1:] if len(r) == len(h)]
    tot = sum(float(r[ist] or 0) for r in data)
    print(kname[:120], "total samples", tot)
    for r in sorted(data, key=lambda r: -float(r[ist] or 0))[:n]:
        print(f"{float(r[ist] or 0) / tot * 100:5.1f}%  {r[ia]:>6}  exec={r[iex]:>10}  {r[isrc][:90]}")
