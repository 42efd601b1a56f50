bash abtest/run2.sh; bash abtest/run2.sh
for L in abtest/lib_base.so abtest/lib_k3g.so abtest/lib_k3g3.so; do GRCA_LIB=$L timeout 300 python bench.py --steps 600 --warmup 10 --no-cpu-baseline --no-hybrid --no-e2e --emulate-world 8 --emulate-rank 7 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N8r7 $L', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms'].items()})"; done
timeout 1400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
