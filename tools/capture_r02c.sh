#!/bin/bash
# ncu --set full captures (summary + per-source-line pages) of the three ladders named in
# DESIGN.md 3b/3c, run under gpurun after the same commands exited 0 in tools/profile_r02c.sh.
cd "$(dirname "$0")/.."
for spec in "td blind_rotate_fft_td 1 tools/run_pbs.py 4096 fft -1 2" "f2td blind_rotate_fft2_td 1 tools/run_pbs_cfg.py CFG4 4096 fft 2" "w blind_rotate_fft_w 2 tools/run_pbs.py 4096 fft -1 1 7"; do
  set -- $spec; k=$1; re=$2; skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o gpurun_out/r02c_ncu_$k python "$@" > gpurun_out/r02c_ncu_$k.log 2>&1
  python profiles/ncu_summary.py gpurun_out/r02c_ncu_$k.ncu-rep > gpurun_out/r02c_ncu_$k.txt 2>&1
  ncu -i gpurun_out/r02c_ncu_$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02c_src_$k.csv 2>/dev/null
  python tools/ncu_smem_lines.py gpurun_out/r02c_src_$k.csv 14 > gpurun_out/r02c_lines_$k.txt; python tools/ncu_lines.py gpurun_out/r02c_src_$k.csv 24 >> gpurun_out/r02c_lines_$k.txt
  rm -f gpurun_out/r02c_ncu_$k.ncu-rep gpurun_out/r02c_src_$k.csv
done
echo captured
