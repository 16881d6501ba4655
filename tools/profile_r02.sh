#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): the bench's PBS step launch list and
# ncu --set full captures of the dominant kernels.  Each ncu command runs only after the
# same command exited 0 without ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --sweep '' --no-other-configs --train-images 0"
eval "$B" > gpurun_out/r02_plain.log 2>&1 && \
  eval "ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $B" \
  > gpurun_out/r02_ncu_launch.log 2>&1
python tools/run_pbs.py 4096 fft -1 1 1 > gpurun_out/r02_plain_tm.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:blind_rotate_fft_tm -s 2 -c 1 \
  -o gpurun_out/r02_ncu_tm python tools/run_pbs.py 4096 fft -1 1 1 > gpurun_out/r02_ncu_tm.log 2>&1
python tools/run_pbs_cfg.py CFG4 4096 fft 1 > gpurun_out/r02_plain_fft2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:blind_rotate_fft2 -s 1 -c 1 \
  -o gpurun_out/r02_ncu_fft2 python tools/run_pbs_cfg.py CFG4 4096 fft 1 > gpurun_out/r02_ncu_fft2.log 2>&1
echo done
