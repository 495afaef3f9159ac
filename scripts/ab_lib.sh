for i in 1 2; do
for v in libflexicache_b200_flat.so libflexicache_b200.so; do
FC_LIB_VARIANT=$v python bench.py --steps 64 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['step_ms']['p50_ms'], d['roofline']['avg_launch_us'], d['roofline']['serialized_launch_us'], d['scored_layer']['us'])" >> gpurun_out/ab.txt
done; done
