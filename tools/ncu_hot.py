"""Top SASS instructions by warp-stall samples from an ncu source-page CSV.
Usage: ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv; python tools/ncu_hot.py s.csv [N] [KERNEL]
A report with several kernels has one "Kernel Name" section each; KERNEL
(0-based, default 0) picks the section."""
import csv, sys
from collections import Counter

_all = list(csv.reader(open(sys.argv[1], errors="replace")))
_sec = [i for i, r in enumerate(_all) if r and r[0] == "Kernel Name"] or [-1]
_pick = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if _pick >= len(_sec):
    sys.exit(f"the report has {len(_sec)} kernel section(s)")
_start = _sec[_pick]
_end = _sec[_pick + 1] if _pick + 1 < len(_sec) else len(_all)
rows = _all[max(_start, 0):_end] if _start >= 0 else [[""]] + _all
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = Counter()
for r in data:
    for h in stall_cols:
        agg[h] += int(r[ix[h]] or 0)
print("total samples", tot)
print("by reason:", ", ".join(f"{h[6:]}={100*v/tot:.1f}%" for h, v in agg.most_common(12)))
# by opcode
op = Counter()
for r in data:
    o = r[ix["Source"]].split()[0] if r[ix["Source"]] else "?"
    if o.startswith("@"):
        o = r[ix["Source"]].split()[1]
    op[o.split(".")[0]] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
print("by opcode:", ", ".join(f"{k}={100*v/tot:.1f}%" for k, v in op.most_common(15)))
data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for r in data[:N]:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:3]
    print(f"{r[ix['Address']]:>8s} {100*s/tot:5.2f}%  {r[ix['Source']][:60]:60s} " + " ".join(f"{n}:{v}" for v, n in top if v))
