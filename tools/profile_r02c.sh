#!/bin/bash
# Round-2 (last session) evidence on one B200 (run under gpurun), after the warp-local
# M <-> B transposes: launch list of the bench's PBS step, ncu --set full of the default
# ladders (cfg2 mode 5, cfg4 N = 2048 TMEM ladder) and of the wide-thread ladder (mode 7).
# Each ncu command runs only after the same command exited 0 without ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --sweep '' --no-other-configs --train-images 0 --infer-images 0 --infer-pbs-images 0 --no-cfg4-full"
eval "$B" > gpurun_out/r02c_plain.log 2>&1 && \
  eval "ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches.csv $B" \
  > gpurun_out/r02c_ncu_launch.log 2>&1
python tools/run_pbs.py 4096 fft -1 2 > gpurun_out/r02c_plain_td.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:blind_rotate_fft_td -s 1 -c 1 \
  -o gpurun_out/r02c_ncu_td python tools/run_pbs.py 4096 fft -1 2 > gpurun_out/r02c_ncu_td.log 2>&1
python tools/run_pbs_cfg.py CFG4 4096 fft 2 > gpurun_out/r02c_plain_f2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:blind_rotate_fft2_td -s 1 -c 1 \
  -o gpurun_out/r02c_ncu_f2td python tools/run_pbs_cfg.py CFG4 4096 fft 2 > gpurun_out/r02c_ncu_f2td.log 2>&1
python tools/run_pbs.py 4096 fft -1 1 7 > gpurun_out/r02c_plain_w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:blind_rotate_fft_w -s 2 -c 1 \
  -o gpurun_out/r02c_ncu_w python tools/run_pbs.py 4096 fft -1 1 7 > gpurun_out/r02c_ncu_w.log 2>&1
# gpurun brings back at most 64 MiB: summarise on the box, keep the per-line source page
for k in td f2td w; do
  python profiles/ncu_summary.py gpurun_out/r02c_ncu_$k.ncu-rep > gpurun_out/r02c_ncu_$k.txt 2>&1
  ncu -i gpurun_out/r02c_ncu_$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02c_src_$k.csv 2>/dev/null
  rm -f gpurun_out/r02c_ncu_$k.ncu-rep
done
echo done
