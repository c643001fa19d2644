#!/bin/bash
# Dev tool: build libvf variants into paper_2209_07632_b200/build/var_<name>.so
# (same sources, -D overrides of one source file), for A/B runs with VF_LIB.
#   tools/variants.sh name:file.cu:-DX=1 ...      (file defaults to vf_device.cu)
set -e
cd "$(dirname "$0")/.."
NVCC=/usr/local/cuda/bin/nvcc
mkdir -p paper_2209_07632_b200/build/var
for spec in "$@"; do
  name=${spec%%:*}; rest=${spec#*:}
  file=${rest%%:*}; defs=${rest#*:}
  case "$file" in *.cu) ;; *) defs=$rest; file=vf_device.cu;; esac
  obj=paper_2209_07632_b200/build/var/${file%.cu}_$name.o
  $NVCC -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-fopenmp,-mavx2,-ffp-contract=off $defs -c paper_2209_07632_b200/csrc/$file -o $obj
  objs=$(ls paper_2209_07632_b200/build/*.o | grep -v "/$file.o")
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2209_07632_b200/build/var_$name.so $objs $obj -lgomp -ldl -lcublas -lcusolver -lcusparse -Xlinker -rpath,/usr/local/cuda/lib64
  echo built $name
done
