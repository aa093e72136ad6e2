"""Stall-reason totals of an ncu source page, overall and for the hot decode region.
  python scripts/ncu_stalls.py REP.ncu-rep"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
iS, iI, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
data = [r for r in rows[1:] if len(r) == len(h)]
def num(x):
    try: return float(x or 0)
    except ValueError: return 0.0
def summary(sel, name):
    tot = sum(num(r[iS]) for r in sel)
    ins = sum(num(r[iI]) for r in sel)
    print(f"== {name}: samples {tot:.0f}, warp-instrs {ins:.0f}")
    agg = {c: sum(num(r[h.index(c)]) for r in sel) for c in reasons}
    for c, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
        print(f"   {c:24s} {v:9.0f} {100*v/max(tot,1):5.1f}%")
summary(data, "all")
# hot region = instructions between the first and last FFMA2 (the unit loops)
idx = [i for i, r in enumerate(data) if "FFMA2" in r[iSrc] or "FMUL2" in r[iSrc]]
if idx:
    summary(data[idx[0]:idx[-1] + 1], f"unit region [{idx[0]}, {idx[-1]}]")
    summary(data[:idx[0]] + data[idx[-1] + 1:], "outside unit region")
print("== top outside-unit instructions by samples (idx samples instrs src)")
outside = [(i, r) for i, r in enumerate(data) if not idx or i < idx[0] or i > idx[-1]]
for i, r in sorted(outside, key=lambda x: -num(x[1][iS]))[:30]:
    print(f"  [{i:5d}] {num(r[iS]):6.0f} {num(r[iI]):10.0f}  {r[iSrc][:80]}")
print("== top by instructions")
for i, r in sorted(outside, key=lambda x: -num(x[1][iI]))[:15]:
    print(f"  [{i:5d}] {num(r[iS]):6.0f} {num(r[iI]):10.0f}  {r[iSrc][:80]}")
