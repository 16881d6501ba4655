#!/bin/bash
# Time cfg3 training and PD-act inference (tools/run_workload.py) for every variants/*.so.
cd "$(dirname "$0")/.."
for so in variants/*.so; do
  echo "== $so"
  for w in train infer; do
    HWB_LIB_PATH=$PWD/$so timeout 300 python tools/run_workload.py $w --cfg ${1:-3} --images 32 --reps 5 2>&1 | tail -1
  done
done
