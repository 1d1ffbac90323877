#!/bin/bash
# A/B the gpuvar/libls_*.so mapped-domain matvec variants (UNITS=geo.cu tools/mv3_variant_libs.sh)
for round in 1 2; do
  for lib in gpuvar/libls_*.so; do
    timeout 300 python -c "
import sys, runpy
import paper_1809_10026_b200 as ls
ls.load_library('$lib')
sys.argv = ['geo_bench.py', '--n-el', '32', '48', '64', '--p', '3', '--no-pcg', '--precond', '0']
runpy.run_path('tools/geo_bench.py', run_name='__main__')
" 2>&1 | sed "s|^{|{\"lib\": \"$lib\", |" | grep '^{'
  done
done
