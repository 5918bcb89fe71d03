"""Per-opcode warp instructions and stall samples of one kernel from an ncu
report's SASS source page (usage: ncu_sass_ops.py REPORT KERNEL_REGEX [N])."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, ist, iin, ith = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                                   "Instructions Executed", "Thread Instructions Executed"))
ops = collections.defaultdict(lambda: [0, 0, 0])
for r in rows[2:]:
    if r and r[0] == "Address":
        continue
    if len(r) <= ith or not r[iin].strip().isdigit():
        continue
    src = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip())
    op = src.split()[0] if src else "?"
    op = op.split(".")[0]
    ops[op][0] += int(r[iin] or 0)
    ops[op][1] += int(r[ist] or 0)
    ops[op][2] += int(r[ith] or 0)
ti = sum(v[0] for v in ops.values()) or 1
ts = sum(v[1] for v in ops.values()) or 1
tt = sum(v[2] for v in ops.values()) or 1
print(f"warp inst {ti}, thread inst {tt}, stall samples {ts}")
for op, (i, s, t) in sorted(ops.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{op:12s} inst {100*i/ti:5.1f}%  thread {100*t/tt:5.1f}%  stall {100*s/ts:5.1f}%")
