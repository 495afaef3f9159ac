#!/bin/bash
# Re-measure the lines the compact owner select affects (profiling aid).
mkdir -p gpurun_out/rb
python bench.py --phases staggered --no-cpu-baseline > gpurun_out/rb/bench_config2_staggered.log 2>&1
FC_PROFILE=spread python bench.py --no-cpu-baseline > gpurun_out/rb/bench_config2_spread.log 2>&1
python bench.py --config 3 > gpurun_out/rb/bench_config3.log 2>&1
python bench.py --serve > gpurun_out/rb/serve.log 2>&1
python bench.py --serve --tiered --query-rho 0.99 > gpurun_out/rb/serve_tiered.log 2>&1
