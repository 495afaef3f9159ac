#!/bin/bash
# The round's measurement set (profiling aid): every bench line this round reports.
set -x
mkdir -p gpurun_out/rb
python -m pytest tests -m gpu -q > gpurun_out/rb/gputest.log 2>&1
python bench.py > gpurun_out/rb/bench_config2.log 2>&1
python bench.py --phases staggered --no-cpu-baseline > gpurun_out/rb/bench_config2_staggered.log 2>&1
FC_PROFILE=spread python bench.py --no-cpu-baseline > gpurun_out/rb/bench_config2_spread.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/rb/bench_reference.log 2>&1
python bench.py --config 3 > gpurun_out/rb/bench_config3.log 2>&1
python bench.py --config 4 --no-cpu-baseline > gpurun_out/rb/bench_config4.log 2>&1
python bench.py --config 5 > gpurun_out/rb/bench_config5.log 2>&1
python bench.py --serve > gpurun_out/rb/serve.log 2>&1
python bench.py --serve --tiered --query-rho 0.99 > gpurun_out/rb/serve_tiered.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/rb/smoke.log 2>&1
