#!/bin/bash
# Builds the standalone B200 measurement tools from source (binaries are not committed).
set -e
cd "$(dirname "$0")"
for t in h2d_sizes hbm_peaks; do
  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o "$t" "$t.cu"
done
