#!/bin/bash
# Build libcmgb variants that differ only in the JVP kernel's tuning macros
# (developer tool): tools/jvp_variants.sh NAME "-DCMGB_JVP_ND=4 ..." [...]
# Output: build/variants/libcmgb_NAME.so (copy over paper_2602_20304_b200/libcmgb.so to A/B).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2602_20304_b200/csrc
B=$ROOT/paper_2602_20304_b200/build
mkdir -p $ROOT/build/variants
make -s -C $CS >/dev/null
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  (
    nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v \
      $flags -c $CS/kernels/manifold_jvp.cu -o $ROOT/build/variants/jvp_$name.o 2> $ROOT/build/variants/jvp_$name.log
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $ROOT/build/variants/libcmgb_$name.so \
      $B/manifold.cu.o $ROOT/build/variants/jvp_$name.o $B/witness.cu.o $B/probe.cu.o $B/api.o $B/mesh_ingest.o \
      $B/sdf_program.o -Xlinker -z,defs -lpthread -ldl -lrt
    echo "$name: $(grep -E 'Used' $ROOT/build/variants/jvp_$name.log | head -1)"
  ) &
done
wait
