#!/bin/bash
# Round-2 profile bundle (run on the GPU box from the repo root): launch lists
# (config 2, config 2 spread, config 4) and full captures of the attention,
# fused-scored and balanced (spread / partial) launches.  Outputs under gpurun_out/prof2/.
set -x
mkdir -p gpurun_out/prof2
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none -k regex:"attn_kernel|score_|step_advance" -c 400 --csv \
  $B > gpurun_out/prof2/launches_config2.csv 2> gpurun_out/prof2/ncu1.err
FC_PROFILE=spread timeout 600 ncu --metrics $M --clock-control none -k regex:"attn|score_|step_advance" -c 400 --csv \
  $B > gpurun_out/prof2/launches_config2_spread.csv 2>> gpurun_out/prof2/ncu1.err
timeout 900 ncu --metrics $M --clock-control none -k regex:"attn|score_|step_advance" -c 300 --csv \
  $B --config 4 > gpurun_out/prof2/launches_config4.csv 2>> gpurun_out/prof2/ncu1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 40 -c 1 \
  -o gpurun_out/prof2/attn $B > /dev/null 2> gpurun_out/prof2/ncu2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_attend_kernel -s 8 -c 1 \
  -o gpurun_out/prof2/score_attend $B > /dev/null 2>> gpurun_out/prof2/ncu2.err
FC_PROFILE=spread timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_attend_bal -s 40 -c 1 \
  -o gpurun_out/prof2/balanced_spread $B > /dev/null 2>> gpurun_out/prof2/ncu2.err
ls -la gpurun_out/prof2
