#!/usr/bin/env bash
# Size-dependent HBM read ceiling on one B200: TMA (2-D boxes, 1-D bulk) and LDG.128 streams of a
# rows x 768-byte matrix (the int8 C2 row) from 7.7 MB to 768 MB, one CTA set per SM, no math.
# scripts/tma_mb is built from scripts/tma_microbench.cu (nvcc -gencode arch=compute_100a,code=sm_100a).
# Output: gpurun_out/read_ceiling.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rows in 10000 30000 100000 300000 1000000; do
  echo "== rows=$rows x 768 B = $(python -c "print(round($rows*768/1e6,1))") MB"
  timeout 120 ./scripts/tma_mb 384 $rows 2>&1 | grep -v '^status'
done > gpurun_out/read_ceiling.txt 2>&1
