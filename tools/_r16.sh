set -x
O=gpurun_out/r16; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_large.py -q -s -p no:cacheprovider -k "c4" > $O/tests.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --config c4 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
grep -n "C4\|passed\|failed\|Error" $O/tests.log | head; python -c "
import json;d=json.loads(open('$O/bench_c4.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['config']['tol'],d['quality'],[(k,round(v['us']/1000,1)) for k,v in d['kernel_shares'].items()])"
