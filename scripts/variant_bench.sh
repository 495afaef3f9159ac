#!/bin/bash
# per-kernel timings (scripts/kernel_bench.py) for library variants in build/
for v in "$@"; do
  cp build/lib_$v.so paper_2511_00868_b200/libflexicache_b200.so
  echo "== $v $(timeout 300 python scripts/kernel_bench.py 2>&1 | tail -1)"
done
