#!/bin/bash
# A/B measurement of kernel build variants: build each -D flag set into
# variants/<name>.so here (nvcc cross-compiles), then on the GPU box run
#   tools/ab_variants.sh run [B ...]
# which times cfg2 PBS batches in both ladder modes for every variants/*.so.
#   tools/ab_variants.sh build name "-DFLAG=1 -DOTHER=0" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
if [ "$1" = build ]; then
  shift
  mkdir -p variants
  while [ $# -ge 2 ]; do
    name=$1; flags=$2; shift 2
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 $flags \
      -Xcompiler -fPIC -shared -o variants/$name.so paper_2403_20190_b200/csrc/hwb_kernels.cu 2>&1 | grep -i error || true
    echo "built variants/$name.so ($flags)"
  done
elif [ "$1" = run ]; then
  shift
  for so in variants/*.so; do
    echo "== $so"
    HWB_LIB_PATH=$PWD/$so timeout 300 python tools/lat_sweep.py "$@" 2>&1 | tail -n $#
  done
fi
