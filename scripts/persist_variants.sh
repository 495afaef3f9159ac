#!/bin/bash
# persistent-kernel library variants (build/lib_<name>.so): run_probe at the
# given batches plus config 3 / config 4-share bench lines; profiling aid
for v in "$@"; do
  cp build/lib_$v.so paper_2511_00868_b200/libflexicache_b200.so
  for b in 1 8; do echo "== $v B=$b $(B=$b SKIP_RUN= timeout 300 python scripts/run_probe.py 2>&1 | tail -1)"; done
  echo "== $v c4 $(timeout 600 python bench.py --config 4 --steps 32 --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])')"
done
