#!/bin/bash
# Build an experimental variant of the library: tools/build_variant.sh NAME -DWFORM_THREADS=384 ...
name=$1; shift
mkdir -p build
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -cudart static \
  -I include "$@" -o build/lib_$name.so paper_2106_09382_b200/csrc/{pcd_wform,pcd_qblock,pcd_qblock_cw4,pcd_qblock_cw8,pcd_exact,gram,diag,datagen,capi}.cu -Xptxas -v 2>&1 \
  | grep -A2 "Function properties for _ZN7concord16pcd" | tail -1
