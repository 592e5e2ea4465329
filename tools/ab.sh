#!/usr/bin/env bash
# A/B the library variants in scratch/variants on the GPU box: tools/ab.sh "v1 v2 ..." [diag args]
mkdir -p gpurun_out
cp paper_1311_2661_b200/libthetis.so /tmp/libthetis_build.so
vs=$1; shift
for rep in 1 2; do
  for v in $vs; do
    cp scratch/variants/libthetis_$v.so paper_1311_2661_b200/libthetis.so
    echo "$v $(python tools/diag_rows.py "$@" 2>&1 | tail -1)"
  done
done
cp /tmp/libthetis_build.so paper_1311_2661_b200/libthetis.so
