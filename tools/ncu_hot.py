"""Opcode mix and top stall sites of one kernel from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0   # e.g. rows / 32 -> per warp-row
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r != hdr and r[0] != hdr[0]]
agg, st = collections.Counter(), collections.Counter()
for d in data:
    src = re.sub(r"^@!?U?P\w+\s+", "", d["Source"].strip())
    op = (src.split()[0] if src else "?").split(".")[0]
    agg[op] += int(d["Instructions Executed"])
    st[op] += int(d["Warp Stall Sampling (All Samples)"])
tot, ts = sum(agg.values()), sum(st.values())
print("warp instructions", tot, "per unit %.1f" % (tot / units))
for op, c in agg.most_common(24):
    print(op.ljust(12), "%5.1f%%" % (100 * c / tot), "per unit %6.2f" % (c / units), "stall %5.1f%%" % (100 * st[op] / ts))
print()
for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"]))[:30]:
    print(d["Address"][-5:], d["Source"][:64].ljust(64), d["Warp Stall Sampling (All Samples)"], d["Instructions Executed"])
