#!/usr/bin/env bash
# GPU box: quick iteration on THETIS_MODE_ASYNC -- parity subset, a short bench, the launch list of a
# 3-epoch solve on R-MAT 26 (setup kernels included)
set -uo pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "${QUICK_TESTS:-async or alm or config}" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err || tail -5 gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('step', d['ms_per_step'], 'epoch', d['epoch']['ms_median'], d['epoch']['ms_first'], 'frac', d['roofline']['frac']); print(d['result']); print({k:(v['epoch_ms_median'], v['f_beta']) for k,v in d['variants'].items()})"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/launches_diag.csv python tools/diag_rows.py --epochs 3 > gpurun_out/ncu_diag.log 2>&1
python tools/ncu_agg.py gpurun_out/launches_diag.csv 2>&1 | tail -30
