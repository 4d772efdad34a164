"""Per-kernel registers / spills from `nvcc -Xptxas -v` output (stdin): one line per entry."""
import re
import subprocess
import sys

name = None
props = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        props = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name and props == name:
        rows.setdefault(name, {})["spill"] = (int(m.group(2)), int(m.group(3)))
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        rows.setdefault(name, {})["regs"] = int(m.group(1))
dem = subprocess.run(["c++filt"], input="\n".join(rows), capture_output=True, text=True).stdout.split("\n")
for (k, v), d in zip(rows.items(), dem):
    d = re.sub(r"agcn::\(anonymous namespace\)::", "", d)
    d = re.sub(r"\(.*\)$", "", d)
    print(f"{v.get('regs', '?'):>4} regs  spill st/ld {v.get('spill', ('?', '?'))}  {d}")
