#!/bin/bash
# Build an A/B variant of the library: tools/build_variant.sh NAME "-DHPG_X=1 ..." [tu ...]
# -> paper_2412_13733_b200/libhpg_b200_NAME.so (HPG_LIB selects it; tools/gpu_bench_ab.sh).
# Only the listed translation units (default: all) are recompiled with the flags;
# the others are taken from build/.
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2; shift 2 || true
tus=${@:-$(cd paper_2412_13733_b200/csrc && ls *.cu | sed 's/\.cu$//')}
make -j8 > /dev/null
out=/tmp/hpg_build/v_$name; mkdir -p $out; cp build/*.o $out/
for t in $tus; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v $flags \
    -c -o $out/$t.o paper_2412_13733_b200/csrc/$t.cu 2> $out/$t.ptxas.log &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2412_13733_b200/libhpg_b200_$name.so $out/*.o
echo built paper_2412_13733_b200/libhpg_b200_$name.so
