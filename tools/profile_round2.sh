#!/usr/bin/env bash
# Round-2 profile set (GPU box, from the repo root; summaries are built on the CPU side with
# tools/ncu_report.py):
#   1. the default bench line, plain                          -> gpurun_out/bench.json
#   2. the reference arm (oracle on the host)                 -> gpurun_out/bench_ref.json
#   3. the launch list of one bench step (gpu__time_duration) -> gpurun_out/launches.csv
#   4. ncu --set full of one k_async_pi launch (R-MAT 26)     -> gpurun_out/async_full.ncu-rep
#   5. per-config rates                                       -> gpurun_out/r02_configs.jsonl
set -uo pipefail
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || tail -5 gpurun_out/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err || tail -5 gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
tools/ncu_async.sh > gpurun_out/ncu_async.log 2>&1
python tools/config_rates.py > gpurun_out/r02_configs.jsonl 2> gpurun_out/config_rates.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("step", d["ms_per_step"], "epoch", d["epoch"]["ms_median"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["ms_per_step"])
PY
wc -l gpurun_out/r02_configs.jsonl
