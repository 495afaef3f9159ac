for v in "FC_PROFILE=spread" "FC_PROFILE=spread FC_BALANCED=0" "FC_PROFILE=spread --config 4" "FC_PROFILE=spread FC_BALANCED=0 --config 4" "X=1"; do
  envs=$(echo $v | tr ' ' '\n' | grep = | tr '\n' ' '); args=$(echo $v | tr ' ' '\n' | grep -v = | tr '\n' ' ')
  echo "== $v"; env $envs python bench.py --no-cpu-baseline --no-e2e --steps 64 $args | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['step_ms'])"
done
