#!/bin/bash
# ncu evidence for the small-batch path (run on the GPU box from the repo root):
# launch list of config 3's kernels (B = 1, both tiers) and one full capture
# of the per-head persistent attention kernel.  Outputs under gpurun_out/prof3/.
mkdir -p gpurun_out/prof3
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"attn_persist|score_|rerank|fetch_kernel|stage_|step_advance|offload" -c 400 --csv \
  python bench.py --config 3 --steps 16 --warmup 2 > gpurun_out/prof3/launches_config3.csv 2> gpurun_out/prof3/ncu1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_persist -s 20 -c 1 \
  -o gpurun_out/prof3/persist python bench.py --config 3 --steps 16 --warmup 2 > /dev/null 2> gpurun_out/prof3/ncu2.err
ls -la gpurun_out/prof3
