#!/bin/bash
# Time every variants/*.so build on the cfg2 PBS batch in the given FFT modes
# (tools/ab_modes.py; bit-identity columns are meaningless for timing-only builds).
#   tools/ab_run.sh [B] [modes] [sets]
cd "$(dirname "$0")/.."
for so in variants/*.so; do
  echo "== $so"
  HWB_LIB_PATH=$PWD/$so timeout 300 python tools/ab_modes.py ${1:-4096} ${2:-1,2} ${3:-CFG2} 3 2>&1 | grep -v "^$" | tail -n 4
done
