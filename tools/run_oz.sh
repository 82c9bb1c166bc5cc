# Ozaki RR Gram checks (diagnostics)
exec 2>/dev/null
python tools/bench_gram.py --mode 2 --shapes 500000x324x648,2000000x528x1056,50000x147x294 --profile | grep -v Memset
timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -2
SPB_GRAM=oz timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -4
for g in dmma oz; do SPB_GRAM=$g timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 $g', d['ms_per_step'], d['quality'], [ (k,v['us']) for k,v in list(d['kernel_shares'].items())[:5]])"; done
