#!/bin/bash
# per-layer attention (in-step prefetch mode) and whole-step time for
# library variants in build/ (scripts/build_variant.sh); profiling aid
for v in "$@"; do
  cp build/lib_$v.so paper_2511_00868_b200/libflexicache_b200.so
  echo "== $v $(SKIP_RUN=1 timeout 300 python scripts/run_probe.py 2>&1 | tail -1)"
done
