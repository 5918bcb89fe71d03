"""Registers / spills per kernel from an nvcc -Xptxas=-v log (stdin)."""
import re
import subprocess
import sys

name = None
rows = []
spill = ""
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        spill = f"spill {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        dem = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
        rows.append((dem.split("(")[0], int(m.group(1)), spill))
        name, spill = None, ""
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for n, r, s in rows:
    if pat in n:
        print(f"{r:4d} {s:18s} {n}")
