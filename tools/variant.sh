#!/usr/bin/env bash
# build libthetis.so with extra -D flags into scratch/variants/libthetis_<name>.so (experiments only)
set -euo pipefail
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p scratch/variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I include -I paper_1311_2661_b200/csrc "$@" paper_1311_2661_b200/csrc/*.cu \
  -o scratch/variants/libthetis_$name.so
