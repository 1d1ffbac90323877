#!/bin/bash
# Build libls.so variants that differ only in mv3.cu's tuning macros (matvec v3), for
# A/B runs with tools/ab_mv.py on one box:  bash tools/mv3_variant_libs.sh tag "-DFOO=1" ...
# Output: gpuvar/libls_<tag>.so (the other objects are the in-tree build's).  UNITS="mv2.cu api.cu"
# rebuilds other translation units with the macros instead (default mv3.cu).
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null
NCCL=$(python -c "import nvidia,os;print([os.path.join(p,'nccl') for p in nvidia.__path__][0])")
B=paper_1809_10026_b200/build
mkdir -p gpuvar
tag=$1; shift
UNITS=${UNITS:-mv3.cu}
objs=$(ls $B/*.o)
vobjs=""
for u in $UNITS; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
    "$@" -I include -I paper_1809_10026_b200/csrc -I $NCCL/include \
    -c paper_1809_10026_b200/csrc/$u -o gpuvar/${u}_$tag.o
  objs=$(echo "$objs" | grep -v "/$u.o$")
  vobjs="$vobjs gpuvar/${u}_$tag.o"
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o gpuvar/libls_$tag.so \
  $objs $vobjs -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
echo gpuvar/libls_$tag.so
