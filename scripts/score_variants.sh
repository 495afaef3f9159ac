#!/bin/bash
# spread-profile scored-layer timings for library variants (profiling aid)
for v in "$@"; do
  cp build/lib_$v.so paper_2511_00868_b200/libflexicache_b200.so
  echo "== $v"; timeout 300 python scripts/spread_probe.py 2>&1 | tail -1
done
cp build/lib_base.so paper_2511_00868_b200/libflexicache_b200.so
