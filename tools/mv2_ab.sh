#!/bin/bash
# A/B the gpuvar/libls_*.so matvec-v2 variants (UNITS="mv2.cu api.cu" tools/mv3_variant_libs.sh)
for round in 1 2; do
  for cfg in 5:2; do
    for lib in gpuvar/libls_*.so; do
      timeout 300 python tools/ab_mv.py $lib $cfg 2 2>&1 | tail -1
    done
  done
done
