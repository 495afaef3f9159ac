#!/bin/bash
# time score / score+select for library variants (profiling aid)
for v in "$@"; do
  cp build/lib_$v.so paper_2511_00868_b200/libflexicache_b200.so
  echo "== $v"; L=2 timeout 300 python scripts/attn_probe.py 2>&1 | grep score_select_us | cut -c1-300
done
