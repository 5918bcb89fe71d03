"""Per CUDA source line: warp-stall samples and instructions executed, from an
ncu report's source page (usage: ncu_src_stalls.py REPORT KERNEL_REGEX [N])."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = None
hdr = None
for line in out.splitlines():
    r = next(csv.reader(io.StringIO(line)), [])
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and len(r) >= 8:  # a CUDA source line (SASS rows have an empty line no)
        try:
            st = int(r[4] or 0)
            ins = int(r[7] or 0)
        except ValueError:
            continue
        if st or ins:
            rows.append((st, ins, fname, r[0], r[1].strip()))
tot_s = sum(x[0] for x in rows) or 1
tot_i = sum(x[1] for x in rows) or 1
print(f"stall samples {tot_s}, warp instructions {tot_i}")
for st, ins, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*st/tot_s:5.1f}% stall {100*ins/tot_i:5.1f}% inst  {f}:{ln}  {src[:80]}")
