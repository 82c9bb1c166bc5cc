O=gpurun_out/chk; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_gram.py -x -q -s -p no:cacheprovider > $O/t_large.log 2>&1; grep -E 'C3|C4|passed|failed|Error' $O/t_large.log | head -20
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; python - <<'P'
import json; d=json.load(open('gpurun_out/chk/bench.json')); r=d['roofline']
print(d['ms_per_step'], d['value'], d['e2e']['value'], r['kernel'], r['frac'], d['step_ms'])
print({k:(v['us'],v['launches']) for k,v in d['kernel_shares'].items()})
P
