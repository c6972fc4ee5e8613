"""Print the hottest SASS lines of an ncu source-page CSV (sass view)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
iS = h.index("Warp Stall Sampling (All Samples)"); iSrc = h.index("Source"); iE = h.index("Instructions Executed")
iT = h.index("Thread Instructions Executed")
tot = sum(float(r[iS] or 0) for r in data)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
# opcode histogram weighted by executed instructions
from collections import Counter
ops = Counter(); samp = Counter()
for r in data:
    op = r[iSrc].split()[0] if r[iSrc].split() else "?"
    if op.startswith("@"): op = r[iSrc].split()[1]
    op = op.split(".")[0]
    ops[op] += float(r[iE] or 0); samp[op] += float(r[iS] or 0)
te = sum(ops.values())
print("opcode mix (warp-inst %, stall-sample %):")
for op, c in ops.most_common(25):
    print(f"  {op:10s} {100*c/te:6.2f}% {100*samp[op]/tot:6.2f}%")
print("hottest lines:")
extra = [h.index(c) for c in ("stall_long_sb", "stall_wait", "stall_branch_resolving") if c in h]
for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:n]:
    print(f"  {100*float(r[iS] or 0)/tot:5.2f}% {r[0]} {r[iSrc][:70]:70s} thr/inst={float(r[iT] or 0)/max(float(r[iE] or 1),1):.1f} " +
          " ".join(h[i][6:] + "=" + r[i] for i in extra))
