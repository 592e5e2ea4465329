"""Per-kernel averages of an ncu --csv metrics log (tools/profile_round.sh step 3)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    agg[d["Kernel Name"][:48]][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
for k, v in agg.items():
    n = len(v["gpu__time_duration.sum"])
    out = []
    for m, x in sorted(v.items()):
        a = sum(x) / len(x)
        if "time" in m:
            out.append("ms %.3f" % (a / 1e6))
        elif "bytes" in m:
            out.append("%s %.3f GB" % (m.split("__")[1].split(".")[0], a / 1e9))
        else:
            out.append("%s %.1f" % (m.split("__")[-1], a))
    print(k.ljust(48), n, " ".join(out))
