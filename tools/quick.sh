#!/usr/bin/env bash
# quick GPU iteration: build, the config-5/2 parity tests, epoch timing, per-kernel DRAM bytes
set -uo pipefail
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests/test_configs_gpu.py tests/test_parity_gpu.py -q -x -k "${QUICK_TESTS:-config5 or config2 or async}" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b.json')); print('step', d['ms_per_step'], 'epoch', d['epoch']['ms_median'], d['epoch']['ms_first'], 'f', d['result']['f_beta'])"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"${QUICK_KERNELS:-k_async|k_hub|k_rows|k_slack}" --csv --log-file gpurun_out/dram.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_dram.log 2>&1
python tools/ncu_agg.py gpurun_out/dram.csv
