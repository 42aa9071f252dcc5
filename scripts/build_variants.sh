#!/bin/bash
# Build libsdfgi_b200.so variants with different -D knobs into paper_2007_14394_b200/_variants/
# usage: scripts/build_variants.sh NAME "-DFOO=1 -DBAR=2" [NAME2 "FLAGS2" ...]
set -e
cd "$(dirname "$0")/.."
P=paper_2007_14394_b200
OUT=$P/_variants
mkdir -p $OUT
F32FLAGS=${F32FLAGS--prec-sqrt=false -prec-div=false -ftz=true}
COMMON="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include"
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p $OUT/$name
  nvcc $COMMON $flags -fmad=false -c $P/csrc/kernels_f64.cu -o $OUT/$name/f64.o &
  nvcc $COMMON $flags -fmad=true $F32FLAGS -c $P/csrc/kernels_f32.cu -o $OUT/$name/f32.o &
  nvcc $COMMON $flags -c $P/csrc/sdfgi_abi.cu -o $OUT/$name/abi.o &
  nvcc $COMMON $flags -c $P/csrc/fp_peak.cu -o $OUT/$name/fp.o &
  nvcc $COMMON $flags -fmad=false -c $P/csrc/select.cu -o $OUT/$name/select.o &
  g++ -std=c++17 -fPIC -fvisibility=hidden -pthread -O2 -ffp-contract=off -fno-fast-math -c $P/csrc/host_trig.cpp -o $OUT/$name/host_trig.o &
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$name/libsdfgi_b200.so $OUT/$name/*.o -lnccl -lcudart -Xcompiler -pthread
  echo built $OUT/$name
done
