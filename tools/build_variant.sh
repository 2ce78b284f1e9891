#!/bin/bash
# Build an experimental libhlbm variant into variants/<name>/libhlbm.so with extra nvcc flags
# (e.g. tools/build_variant.sh s2 -DHLBM_F32_STAGES=1 -DHLBM_F32_NB=2); select it with HLBM_LIB.
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2602_05295_b200/csrc"
out=../../variants/$name; mkdir -p $out
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC"
objs=""
for f in hlbm_interior hlbm_interior_q0 hlbm_interior_q1 hlbm_interior_q2 hlbm_interior_q19 hlbm_interior_q19m hlbm_cells hlbm_pull_f32 hlbm_pull_q16 hlbm_alg1 hlbm_mesh hlbm_capi; do
  nvcc $FL "$@" -c $f.cu -o $out/$f.o & objs="$objs $out/$f.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libhlbm.so $objs -lcudart
echo built $out/libhlbm.so
