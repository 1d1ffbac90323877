#!/bin/bash
# A/B the gpuvar/libls_*.so matvec-v3 variants (tools/mv3_variant_libs.sh): two interleaved rounds.
mkdir -p gpurun_out
for round in 1 2; do
  for cfg in 4 5:8 5:4; do
    for lib in gpuvar/libls_*.so; do
      timeout 300 python tools/ab_mv.py $lib $cfg 3 2>&1 | tail -1
    done
  done
done
