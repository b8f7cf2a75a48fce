#!/bin/bash
# Build the standalone timing probes (not part of the library).
cd "$(dirname "$0")" && for f in chol_probe lat_probe d2_probe df_probe pdl_probe bar_probe read_probe; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -w $f.cu -o $f || exit 1
done
