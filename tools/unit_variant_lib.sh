#!/bin/bash
# Build a libls.so variant in which ONE translation unit (e.g. ft.cu) is recompiled with extra
# tuning macros; every other object is the in-tree build's.  For A/B runs on one box:
#   bash tools/unit_variant_lib.sh tag ft.cu "-DLS_FT_D=8" ...   -> gpuvar/libls_<tag>.so
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null
NCCL=$(python -c "import nvidia,os;print([os.path.join(p,'nccl') for p in nvidia.__path__][0])")
B=paper_1809_10026_b200/build
mkdir -p gpuvar
tag=$1; unit=$2; shift 2
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
  "$@" -I include -I paper_1809_10026_b200/csrc -I $NCCL/include \
  -c paper_1809_10026_b200/csrc/$unit -o gpuvar/${unit}_$tag.o
objs=""
for o in $B/*.o; do
  if [ "$(basename $o)" = "$unit.o" ]; then objs="$objs gpuvar/${unit}_$tag.o"; else objs="$objs $o"; fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o gpuvar/libls_$tag.so \
  $objs -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
echo gpuvar/libls_$tag.so
