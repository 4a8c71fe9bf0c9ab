"""Registers and spill bytes per kernel from the ptxas -v output in _lib/build.log."""
import re
import subprocess
import sys

log = sys.argv[1] if len(sys.argv) > 1 else "paper_2010_13972_b200/_lib/build.log"
fn = None
rows = {}
for line in open(log):
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        fn = m.group(1)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and fn:
        rows.setdefault(fn, {})["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and fn:
        rows.setdefault(fn, {})["regs"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for n, d in zip(names, dem):
    r = rows[n]
    if "nodal_kernel" in d or "bins" in d or r.get("spill", (0, 0)) != (0, 0):
        print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill')}  {d}")
