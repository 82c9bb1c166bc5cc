# bench A/B (diagnostics): default vs an env switch given as $1
exec 2>/dev/null
timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('default', d['ms_per_step'], [ (k,v['us']) for k,v in list(d['kernel_shares'].items())[:4]])"; done
for i in 1 2; do env $1 timeout 300 python bench.py --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], [ (k,v['us']) for k,v in list(d['kernel_shares'].items())[:4]])"; done
timeout 400 python bench.py --config c3 --steps 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3', d['ms_per_step'], [ (k,v['us']) for k,v in list(d['kernel_shares'].items())[:6]])"
