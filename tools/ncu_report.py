#!/usr/bin/env python
"""Summaries of this round's ncu captures for profiles/ (CPU side, reads gpurun_out/).

  python tools/ncu_report.py launches <launches.csv> <out.txt>
      per-kernel launch counts, device time and share of one bench step
      (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)
  python tools/ncu_report.py full <report.ncu-rep> <out.txt> [--summary profiles/ncu_summary.json]
      one kernel's --set full capture: duration, DRAM bytes, L2 hit and miss by operation,
      RED / ATOM instruction and sector counts, occupancy, issue activity, top stall reasons
      and the SASS lines with most stall samples; --summary also writes the DRAM bytes per
      launch that bench.py reports as roofline.traffic
"""
import collections
import csv
import json
import re
import subprocess
import sys


def short(name):
    m = re.search(r"([A-Za-z_]\w*)(<[^(]*>)?\(", name)
    base = m.group(1) if m else name
    return base if base.startswith("k_") else name.split("(")[0][:70]


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr, data = rows[0], rows[1:]
    iname, ival = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for r in data:
        nm = short(r[iname])
        tot[nm] = tot.get(nm, 0.0) + float(r[ival].replace(",", ""))
        cnt[nm] += 1
    T = sum(tot.values())
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none, one bench step: {sum(cnt.values())} "
             f"launches, {T / 1e6:.2f} ms total (cold-cache and serialised: compare shares, not absolutes)",
             f"{'ms total':>10} {'share':>6} {'launches':>8} {'ms/launch':>10}  kernel"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{v / 1e6:10.3f} {100 * v / T:5.1f}% {cnt[k]:8d} {v / 1e6 / cnt[k]:10.3f}  {k}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:12]))


RAW = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
       ("dram__bytes_write.sum", "DRAM write"), ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
       ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
       ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors"),
       ("lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "L2 read sectors missed"),
       ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 RED sectors"),
       ("lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum", "L2 RED sectors missed"),
       ("lts__t_sectors_srcunit_tex_op_atom.sum", "L2 ATOM sectors"),
       ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 write sectors"),
       ("smsp__inst_executed_op_global_red.sum", "RED instructions (warp)"),
       ("smsp__sass_inst_executed_op_global_ld.sum", "global LD instructions (warp)"),
       ("smsp__inst_executed_op_shared_atom.sum", "shared ATOM instructions (warp)"),
       ("lts__t_sectors_srcunit_ltcfabric.sum", "L2 sectors across the die fabric"),
       ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
       ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
       ("launch__registers_per_thread", "registers / thread"), ("launch__grid_size", "grid"),
       ("launch__block_size", "block")]


def full(rep, out, summary=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    name = short(vals[hdr.index("Kernel Name")]) if "Kernel Name" in hdr else "?"
    lines = [f"# ncu --set full --clock-control none: {name} (one launch)"]
    for key, label in RAW:
        if key in get:
            u, v = get[key]
            lines.append(f"{label:40s} {v} {u}")
    stalls = [(h.split("smsp__average_warp_latency_issue_stalled_")[1].split(".")[0], float(v))
              for h, v in zip(hdr, vals) if h.startswith("smsp__average_warp_latency_issue_stalled_")
              and h.endswith(".ratio") and v not in ("", "n/a")]
    if stalls:
        lines.append("stall reasons (cycles per issued instruction): " +
                     ", ".join(f"{k} {v:.2f}" for k, v in sorted(stalls, key=lambda x: -x[1])[:6]))
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(src.splitlines()))
    if len(srows) > 2:
        sh = srows[1]
        data = [dict(zip(sh, r)) for r in srows[2:] if len(r) == len(sh) and r[0] != sh[0]]
        tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
        lines.append("top SASS lines by stall samples:")
        for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:12]:
            lines.append(f"  {100 * int(d['Warp Stall Sampling (All Samples)']) / tot:5.1f}%  {d['Source'].strip()[:80]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if summary:
        rb = float(get["dram__bytes_read.sum"][1].replace(",", "")) * (1e9 if get["dram__bytes_read.sum"][0] == "Gbyte" else 1)
        wb = float(get["dram__bytes_write.sum"][1].replace(",", "")) * (1e9 if get["dram__bytes_write.sum"][0] == "Gbyte" else 1)
        def num(key):
            return float(get[key][1].replace(",", "")) if key in get and get[key][1] not in ("", "n/a") else None
        json.dump({"kernel": name, "epoch_dram_bytes": rb + wb, "dram_read_bytes": rb, "dram_write_bytes": wb,
                   "l2_read_sectors": num("lts__t_sectors_srcunit_tex_op_read.sum"),
                   "l2_red_sectors": num("lts__t_sectors_srcunit_tex_op_red.sum"),
                   "l2_hit_rate_pct": num("lts__t_sector_hit_rate.pct"),
                   "duration_ms": num("gpu__time_duration.sum"),
                   "source": rep, "note": "dram__bytes_read.sum + dram__bytes_write.sum of one launch (= one epoch); "
                                          "L2 sectors by operation of the same launch"},
                  open(summary, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[5] if len(sys.argv) > 5 and sys.argv[4] == "--summary" else None)
