#!/bin/bash
# Round-2 (second session) evidence on one B200 (run under gpurun): launch list of the
# bench's PBS step, ncu --set full of the default ladders (cfg2 mode 5, cfg4 N = 2048
# TMEM ladder), and DRAM bytes of one cfg2 batch without ncu's cache flush.  Each ncu
# command runs only after the same command exited 0 without ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --sweep '' --no-other-configs --train-images 0 --infer-images 0 --infer-pbs-images 0 --no-cfg4-full"
eval "$B" > gpurun_out/r02b_plain.log 2>&1 && \
  eval "ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches.csv $B" \
  > gpurun_out/r02b_ncu_launch.log 2>&1
python tools/run_pbs.py 4096 fft -1 1 > gpurun_out/r02b_plain_td.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:blind_rotate_fft_td -s 2 -c 1 \
  -o gpurun_out/r02b_ncu_td python tools/run_pbs.py 4096 fft -1 1 > gpurun_out/r02b_ncu_td.log 2>&1
python tools/run_pbs.py 4096 fft -1 1 > /dev/null 2>&1 && \
  ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  -k regex:blind_rotate_fft_td -s 10 -c 10 --csv python tools/run_pbs.py 4096 fft -1 2 > gpurun_out/r02b_noflush_td.csv 2>&1
python tools/run_pbs_cfg.py CFG4 4096 fft 1 > gpurun_out/r02b_plain_f2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:blind_rotate_fft2_td -s 1 -c 1 \
  -o gpurun_out/r02b_ncu_f2td python tools/run_pbs_cfg.py CFG4 4096 fft 1 > gpurun_out/r02b_ncu_f2td.log 2>&1
echo done
