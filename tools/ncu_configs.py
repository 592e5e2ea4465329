#!/usr/bin/env python
"""Summary of tools/ncu_configs.sh (CPU side): per config one mid-run async epoch's DRAM bytes,
sector efficiency (algorithmic bytes / DRAM bytes), L2 hit rate, L2 read / RED sectors and rates.
  python tools/ncu_configs.py gpurun_out profiles/r02_ncu_configs.txt"""
import csv
import json
import os
import sys

src, out = sys.argv[1], sys.argv[2]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
alg = {}
for l in open(os.path.join(ROOT, "profiles", "r02_configs.jsonl")):
    x = json.loads(l)
    alg[x["config"]] = x["alg_bytes_per_epoch"]
lines = ["# ncu --clock-control none, the 6th k_async_pi launch (one epoch) of tools/config_rates.py --modes 1 per config",
         "# (first step rule of the config's runs: 1/L_max).  sector efficiency = algorithmic bytes (20 n_s + 12 nnz_s + 16 m) / DRAM bytes",
         f"{'config':16s} {'ms':>8s} {'DRAM GB':>9s} {'alg GB':>8s} {'sect.eff':>8s} {'L2 hit%':>8s} {'L2 rd sect':>11s} {'L2 RED sect':>11s} "
         f"{'G sect/s':>9s} {'RED inst':>10s} {'occ%':>6s}"]
for c in ("vc_er_1k", "mis_er_1m", "vc_chunglu_10m", "mwc_grid_2048", "vc_rmat_26"):
    p = os.path.join(src, f"ncu_cfg_{c}.csv")
    if not os.path.exists(p):
        continue
    rows = [r for r in csv.reader(open(p)) if len(r) > 5]
    if len(rows) < 2:
        continue
    h = rows[0]
    iname, ival, iunit = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    m = {}
    for r in rows[1:]:
        v = float(r[ival].replace(",", ""))
        u = r[iunit]
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e6, "us": 1e3, "ns": 1, "s": 1e9}.get(u, 1)
        m[r[iname]] = v * scale
    ms = m["gpu__time_duration.sum"] / 1e6
    dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    rd, red = m["lts__t_sectors_srcunit_tex_op_read.sum"], m["lts__t_sectors_srcunit_tex_op_red.sum"]
    lines.append(f"{c:16s} {ms:8.3f} {dram / 1e9:9.3f} {alg[c] / 1e9:8.3f} {alg[c] / max(dram, 1):8.2f} "
                 f"{m['lts__t_sector_hit_rate.pct']:8.1f} {rd:11.3e} {red:11.3e} {(rd + red) / ms / 1e6:9.1f} "
                 f"{m.get('smsp__inst_executed_op_global_red.sum', 0):10.3e} "
                 f"{m.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):6.1f}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
