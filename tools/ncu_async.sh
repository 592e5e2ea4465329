#!/usr/bin/env bash
# GPU box: one --set full capture of the async epoch kernel on the bench workload (R-MAT 26),
# after a plain run of the same command.  Output: gpurun_out/async_full.ncu-rep (+ plain log).
set -uo pipefail
mkdir -p gpurun_out
python tools/diag_rows.py --epochs 4 ${DIAG_ARGS:-} > gpurun_out/diag_plain.json 2> gpurun_out/diag_plain.err || { tail -5 gpurun_out/diag_plain.err; exit 1; }
cat gpurun_out/diag_plain.json
ncu --set full --clock-control none --import-source on -k regex:k_async_pi --launch-skip 2 --launch-count 1 \
    -o gpurun_out/async_full -f python tools/diag_rows.py --epochs 4 ${DIAG_ARGS:-} > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out/*.ncu-rep
