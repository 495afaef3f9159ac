#!/bin/bash
# Round profile bundle (run on the GPU box from the repo root): bench lines,
# ncu launch list of the bench's kernels, full captures of the attention and
# scoring kernels.  Outputs under gpurun_out/prof/.
set -x
mkdir -p gpurun_out/prof
timeout 400 python bench.py > gpurun_out/prof/bench.jsonl 2> gpurun_out/prof/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/prof/bench_reference.jsonl 2>> gpurun_out/prof/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"attn_kernel|score_|step_advance" -c 400 --csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/launches.csv 2> gpurun_out/prof/ncu1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 40 -c 1 \
  -o gpurun_out/prof/attn python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/prof/ncu2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_attend -s 8 -c 1 \
  -o gpurun_out/prof/score_attend python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2> gpurun_out/prof/ncu3.err
ls -la gpurun_out/prof
