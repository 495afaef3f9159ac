mkdir -p gpurun_out/fix
python -m pytest tests -m gpu -x -q -k "parity or phases or engine" > gpurun_out/fix/tests.log 2>&1; tail -3 gpurun_out/fix/tests.log
for c in 2 4; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-variants 2>/dev/null | tail -1 > gpurun_out/fix/c$c.json; done
FC_PROFILE=spread timeout 600 python bench.py --config 4 --no-cpu-baseline --no-e2e --no-variants 2>/dev/null | tail -1 > gpurun_out/fix/c4s.json
FC_PROFILE=spread timeout 600 python bench.py --config 2 --no-cpu-baseline --no-e2e --no-variants 2>/dev/null | tail -1 > gpurun_out/fix/c2s.json
timeout 600 python bench.py --config 2 --phases staggered --no-cpu-baseline --no-e2e --no-variants 2>/dev/null | tail -1 > gpurun_out/fix/c2p.json
for f in gpurun_out/fix/c*.json; do echo $f; python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d.get('roofline',{}).get('frac'))"; done
