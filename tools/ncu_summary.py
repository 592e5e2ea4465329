#!/usr/bin/env python
"""Summarise the ncu CSVs of tools/profile_round.sh into profiles/ (CPU side).

profiles/<round>_launches.txt : per-kernel launch counts, total / mean device time and
                                 share of one bench step (cold-cache, serialised)
profiles/<round>_epoch_dram.txt: DRAM bytes and L2 hit rate per launch of the epoch kernels
profiles/ncu_summary.json      : what bench.py reads for roofline.traffic (bytes per epoch)
"""
import collections
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    """kernel base name: the identifier right before the argument list"""
    m = re.search(r"([A-Za-z_]\w*)(<[^(]*>)?\(", name)
    base = m.group(1) if m else name
    return base if base.startswith("k_") else name.split("(")[0][:70]


def rows(path):
    out = [r for r in csv.reader(open(path)) if len(r) > 5]
    return out[0], out[1:]


def main(tag, out_dir):
    os.makedirs(out_dir, exist_ok=True)
    hdr, data = rows(os.path.join(ROOT, "gpurun_out", "launches.csv"))
    iname, ival = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for r in data:
        nm = short(r[iname])
        v = float(r[ival].replace(",", ""))
        tot[nm] = tot.get(nm, 0.0) + v
        cnt[nm] += 1
    T = sum(tot.values())
    lines = [f"# {tag}: ncu --metrics gpu__time_duration.sum --clock-control none, one bench step "
             f"(python bench.py --steps 1 --warmup 0), {sum(cnt.values())} launches, {T / 1e6:.2f} ms total",
             "# cold-cache and serialised: compare shares, not absolutes",
             f"{'ms total':>10} {'share':>6} {'launches':>8} {'ms/launch':>10}  kernel"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{v / 1e6:10.3f} {100 * v / T:5.1f}% {cnt[k]:8d} {v / 1e6 / cnt[k]:10.3f}  {k}")
    open(os.path.join(out_dir, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")

    hdr, data = rows(os.path.join(ROOT, "gpurun_out", "dram.csv"))
    iname, imet, ival, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                              hdr.index("ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        per[r[iid]][r[imet]] = float(r[ival].replace(",", ""))
        names[r[iid]] = short(r[iname])
    agg = collections.defaultdict(lambda: collections.Counter())
    for i, m in per.items():
        nm = names[i]
        agg[nm]["launches"] += 1
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            agg[nm][k] += m.get(k, 0.0)
        agg[nm]["hit"] += m.get("lts__t_sector_hit_rate.pct", 0.0)
    lines = [f"# {tag}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
             "lts__t_sector_hit_rate.pct on the epoch kernels of one bench step (20 epochs)",
             f"{'launches':>8} {'GB read':>9} {'GB write':>9} {'ms':>8} {'L2 hit%':>8}  kernel (per launch)"]
    epoch_total = 0.0
    # one k_async (or k_slack_sweep) launch per epoch; kernels launched once per call (the
    # application of the pending hub steps) are spread over the call's epochs
    n_epochs = max([agg[k]["launches"] for k in agg if k.startswith(("k_async", "k_slack"))] or [1])
    for nm, c in sorted(agg.items()):
        n = c["launches"]
        rd, wr = c["dram__bytes_read.sum"] / n, c["dram__bytes_write.sum"] / n
        lines.append(f"{n:8d} {rd / 1e9:9.3f} {wr / 1e9:9.3f} {c['gpu__time_duration.sum'] / n / 1e6:8.3f} "
                     f"{c['hit'] / n:8.1f}  {nm}")
        if nm.startswith(("k_async", "k_hub_update", "k_rows", "k_slack")):
            epoch_total += c["dram__bytes_read.sum"] + c["dram__bytes_write.sum"]
    epoch_bytes = epoch_total / n_epochs
    lines.append(f"# DRAM bytes per epoch (epoch kernels' bytes over {n_epochs} epochs): {epoch_bytes / 1e9:.3f} GB")
    open(os.path.join(out_dir, f"{tag}_epoch_dram.txt"), "w").write("\n".join(lines) + "\n")
    json.dump({"round": tag, "epoch_dram_bytes": epoch_bytes,
               "note": "sum of dram__bytes_read.sum + dram__bytes_write.sum over the kernels of one SCD epoch"},
              open(os.path.join(out_dir, "ncu_summary.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01", os.path.join(ROOT, "profiles"))
