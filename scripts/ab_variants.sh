#!/bin/bash
# Build libphiks variants of ozaki.cu with compile-time experiment switches into
# build_exp/<name>/libphiks.so (A/B timing with PHIKS_LIB_PATH, scripts/ab_step.sh).
# usage: scripts/ab_variants.sh name "-DOZ_DESC=0" [name2 "-D..."] ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2210_07667_b200/csrc
make -C "$CS" -j8 >/dev/null
NVCC=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I$ROOT/include -Xcompiler -fPIC"
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  out=$ROOT/build_exp/$name; mkdir -p "$out"
  $NVCC $FL $defs -c "$CS/ozaki.cu" -o "$out/ozaki.o"
  objs=$(ls $CS/build/*.o | grep -v ozaki.o)
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libphiks.so" $objs "$out/ozaki.o" \
    -cudart static -Xlinker -z,defs -lgomp -lpthread -ldl -lrt
  echo "built $out/libphiks.so ($defs)"
done
