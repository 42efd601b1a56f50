set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "update_scene or indexed or float3 or hybrid or c2_tilted" 2>&1 | tail -5
for a in "" "--soup"; do
  for i in 1 2; do timeout 300 python bench.py --steps 600 --warmup 10 --no-cpu-baseline --no-hybrid $a 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N1[$a]', round(d['ms_per_step'],4), d['e2e']['ms_per_step'] if d.get('e2e') else None, {k: round(v,4) for k,v in d['kernel_ms'].items()})"; done
  timeout 300 python bench.py --steps 600 --warmup 10 --no-cpu-baseline --no-hybrid --no-e2e --emulate-world 8 --emulate-rank 7 $a 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N8r7[$a]', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms'].items()})"
done
