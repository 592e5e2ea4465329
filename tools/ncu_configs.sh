#!/usr/bin/env bash
# GPU box: one mid-run async epoch (k_async_pi, 6th launch) of every BASELINE config under ncu:
# DRAM bytes, L2 hit rate, L2 read / RED sectors, duration (SURVEY 8(d) "Timing, GPU").
# Output: gpurun_out/ncu_cfg_<config>.csv; summarised by tools/ncu_configs.py.
set -uo pipefail
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
M=$M,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum
M=$M,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum
M=$M,smsp__inst_executed_op_global_red.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for c in vc_er_1k mis_er_1m vc_chunglu_10m mwc_grid_2048 vc_rmat_26; do
  ncu --metrics $M --clock-control none -k regex:k_async_pi --launch-skip 5 --launch-count 1 --csv \
      --log-file gpurun_out/ncu_cfg_$c.csv python tools/config_rates.py --only $c --modes 1 > gpurun_out/ncu_cfg_$c.log 2>&1
  echo "$c done"
done
