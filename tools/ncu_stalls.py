"""Stall-reason totals and the top stalled SASS lines (with their reasons) of one kernel
from `ncu --page source --csv --print-source sass` (experiments only)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[0] != hdr[0]]
seen, uniq = set(), []
for d in data:
    if d["Address"] not in seen:
        seen.add(d["Address"]); uniq.append(d)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for d in uniq:
    for r in reasons:
        tot[r] += int(d[r] or 0)
T = sum(tot.values())
print("stall totals:", ", ".join("%s %.1f%%" % (r[6:], 100 * v / T) for r, v in tot.most_common(8)))
for d in sorted(uniq, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    top = sorted(((int(d[r] or 0), r[6:]) for r in reasons), reverse=True)[:2]
    print(d["Address"][-5:], d["Source"][:56].ljust(56), d["Warp Stall Sampling (All Samples)"].rjust(6),
          " ".join("%s:%d" % (n, v) for v, n in top))
