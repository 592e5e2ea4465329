#!/usr/bin/env bash
# Run on the GPU box (via gpurun) from the repo root:
#   1. the default bench line (plain, no profiler)            -> gpurun_out/bench.json
#   2. the launch list of one bench step (gpu__time_duration) -> gpurun_out/launches.csv
#   3. DRAM bytes of the epoch kernels (one step)             -> gpurun_out/dram.csv
# Summaries are then built on the CPU side with tools/ncu_summary.py.
set -euo pipefail
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/plain_step.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"k_async|k_hub|k_rows|k_slack" --csv --log-file gpurun_out/dram.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_dram.log 2>&1
echo done
