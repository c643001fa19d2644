#!/bin/bash
# Dev tool: build libvf variants of the hot kernel's staging parameters into
# build/var_<name>.so (same sources, -D overrides), for A/B runs with VF_LIB.
set -e
cd "$(dirname "$0")/.."
NVCC=/usr/local/cuda/bin/nvcc
mkdir -p paper_2209_07632_b200/build/var
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  obj=paper_2209_07632_b200/build/var/vf_device_$name.o
  $NVCC -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-fopenmp,-mavx2,-ffp-contract=off $defs -c paper_2209_07632_b200/csrc/vf_device.cu -o $obj
  objs=$(ls paper_2209_07632_b200/build/*.o | grep -v vf_device.cu.o)
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2209_07632_b200/build/var_$name.so $objs $obj -lgomp -ldl -lcublas -lcusolver -lcusparse -Xlinker -rpath,/usr/local/cuda/lib64
  echo built $name
done
