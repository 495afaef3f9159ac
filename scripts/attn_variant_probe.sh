#!/bin/bash
# time the attention kernel for library variants (profiling aid)
for v in "$@"; do
  cp build/lib_$v.so paper_2511_00868_b200/libflexicache_b200.so
  echo "== $v"; L=4 timeout 300 python scripts/attn_probe.py 2>&1 | head -2 | cut -c1-600
done
