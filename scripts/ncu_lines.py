import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
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
        if body: break
        continue
    body.append(r)
tot = sum(int(r[iI] or 0) for r in body)
print("total inst", tot)
# group consecutive lines with equal exec count
cur=None; acc=0; n=0; first=0
for k,r in enumerate(body):
    c=int(r[iI] or 0)
    if c!=cur:
        if cur is not None and acc>0.003*tot: print(f"lines {first:4d}-{k-1:4d} n={n:3d} exec/line={cur:>9} sum={acc/tot*100:5.1f}%  {body[first][iS].strip()[:50]}")
        cur=c; acc=0; n=0; first=k
    acc+=c; n+=1
print(f"lines {first}- n={n} exec={cur} sum={acc/tot*100:.1f}%")
