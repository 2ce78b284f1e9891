#!/bin/bash
# Fast experimental variant: rebuild only the fp32 / default-codec q16 interior units with extra nvcc
# flags, link them with the other objects of the main build (make -C paper_2602_05295_b200/csrc first).
#   tools/build_variant_fast.sh <name> -DFLAG=... ; select with HLBM_LIB=variants/<name>/libhlbm.so
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2602_05295_b200/csrc"
out=../../variants/$name; mkdir -p $out
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC"
nvcc $FL "$@" -c hlbm_interior.cu -o $out/hlbm_interior.o &
nvcc $FL "$@" -c hlbm_interior_q2.cu -o $out/hlbm_interior_q2.o &
wait
objs="$out/hlbm_interior.o $out/hlbm_interior_q2.o"
for f in hlbm_interior_q0 hlbm_interior_q1 hlbm_interior_q19 hlbm_interior_q19m hlbm_cells hlbm_pull_f32 hlbm_pull_q16 hlbm_alg1 hlbm_mesh hlbm_capi; do objs="$objs build/$f.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libhlbm.so $objs -lcudart
rm -f $out/*.o
echo built $out/libhlbm.so
