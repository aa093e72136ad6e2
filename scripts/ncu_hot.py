"""Summarise an ncu source page (SASS): stall samples and executed instructions per region."""
import csv, sys, re, subprocess
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(lines[1:]))
h = rows[0]
iS, iI, iSrc, iA = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source"), h.index("Address")
data = [(int(r[iS] or 0), int(r[iI] or 0), r[iSrc].strip(), r[iA]) for r in rows[1:] if len(r) > iI]
tot_s = sum(d[0] for d in data); tot_i = sum(d[1] for d in data)
print(f"total samples {tot_s}, instructions {tot_i}")
ops = {}
for s, i, src, a in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    op = op.split(".")[0]
    o = ops.setdefault(op, [0, 0]); o[0] += s; o[1] += i
print("by opcode (samples, instrs):")
for op, (s, i) in sorted(ops.items(), key=lambda x: -x[1][0])[:25]:
    print(f"  {op:10s} {s:7d} ({100*s/max(tot_s,1):5.1f}%)  {i:9d} ({100*i/max(tot_i,1):5.1f}%)")
print("hottest instructions:")
for idx, (s, i, src, a) in sorted(enumerate(data), key=lambda x: -x[1][0])[:top]:
    print(f"  [{idx:5d}] {s:6d} {i:8d}  {src[:90]}")
