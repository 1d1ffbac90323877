#!/bin/bash
# Build libls.so variants that differ only in the register-direct FD kernel's tuning macros
# (rd_inst.cu buckets, e.g. -DLS_RD_CS_NT=1 -DLS_RD_CS_MINB=2 -DLS_RD_CS_D=8), for A/B runs
# with tools/ab_fd.py on one box:  bash tools/rd_variant_libs.sh tag "-DFOO=1" ...
# Output: gpuvar/libls_<tag>.so (the other objects are the in-tree build's).
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /dev/null
NCCL=$(python -c "import nvidia,os;print([os.path.join(p,'nccl') for p in nvidia.__path__][0])")
B=paper_1809_10026_b200/build
mkdir -p gpuvar
tag=$1; shift
objs=""
pids=""
for o in $B/*.o; do
  base=$(basename $o)
  case $base in
    rd_ks*.o)
      K=${base#rd_ks}; K=${K%.o}
      /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
        "$@" -DLS_RD_KS=$K -I include -I paper_1809_10026_b200/csrc -I $NCCL/include \
        -c paper_1809_10026_b200/csrc/rd_inst.cu -o gpuvar/rd_ks${K}_$tag.o &
      pids="$pids $!"
      objs="$objs gpuvar/rd_ks${K}_$tag.o";;
    *) objs="$objs $o";;
  esac
done
for p in $pids; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o gpuvar/libls_$tag.so \
  $objs -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
echo gpuvar/libls_$tag.so
