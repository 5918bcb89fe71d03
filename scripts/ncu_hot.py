"""Top SASS lines by warp-stall samples for one kernel of an ncu report."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
iS, iA, iI = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
body = []
for r in rows[1:]:
    if len(r) != len(hdr) or not r[iA].isdigit():
        if body: break   # first kernel instance only
        continue
    body.append(r)
tot = sum(int(r[iA] or 0) for r in body)
print("total samples", tot, "sass lines", len(body))
for k, r in enumerate(body):
    r.append(k)
top = sorted(body, key=lambda r: -int(r[iA] or 0))[:n]
for r in sorted(top, key=lambda r: r[-1]):
    print(f"{r[-1]:5d} {int(r[iA])/tot*100:5.1f}% {r[iI]:>9} {r[iS].strip()[:90]}")
