#!/bin/bash
# compute-sanitizer over the round-2 paths (profiling aid): per-request phases
# and reload pauses, the balanced launch (compact select, bulk score read,
# helper CTAs), the one-CTA recycle, the float64 select, the 2-rank test.
mkdir -p gpurun_out/san2
CS="compute-sanitizer --print-limit 20"
timeout 1200 $CS --tool memcheck python -m pytest -x -q tests/test_gpu_phases.py > gpurun_out/san2/memcheck_phases.log 2>&1
timeout 1200 $CS --tool racecheck python -m pytest -x -q tests/test_gpu_phases.py -k "own_step and bfloat16-128 or holds_only" > gpurun_out/san2/racecheck_phases.log 2>&1
timeout 1200 $CS --tool memcheck python -m pytest -x -q tests/test_gpu_engine.py -k "balanced" > gpurun_out/san2/memcheck_balanced.log 2>&1
timeout 1200 $CS --tool racecheck python -m pytest -x -q tests/test_gpu_engine.py -k "balanced_bitwise" > gpurun_out/san2/racecheck_balanced.log 2>&1
timeout 1200 $CS --tool synccheck python -m pytest -x -q tests/test_gpu_engine.py -k "balanced_bitwise" > gpurun_out/san2/synccheck_balanced.log 2>&1
timeout 1200 $CS --tool memcheck python -m pytest -x -q tests/test_gpu_tiers.py tests/test_gpu_parity.py -k "recycle or select" > gpurun_out/san2/memcheck_recycle_select.log 2>&1
timeout 1200 $CS --tool racecheck python -m pytest -x -q tests/test_gpu_tiers.py -k "recycle" > gpurun_out/san2/racecheck_recycle.log 2>&1
timeout 1200 $CS --tool memcheck python -m pytest -x -q tests/test_gpu_fullsize.py -k "128k and score_mode1" > gpurun_out/san2/memcheck_fullsize_128k.log 2>&1
grep -H -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san2/*.log > gpurun_out/san2/summary.txt
