set -x
O=gpurun_out/r14; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_update.py tests/test_gpu_large.py -q -s -p no:cacheprovider -k "update or c3_partition" > $O/tests.log 2>&1
for a in 0 1; do SPB_UT_ATM=$a timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_atm$a.json 2> $O/bench_atm$a.err; done
tail -3 $O/tests.log; grep -n "C3 \|FAILED" $O/tests.log | head; for a in 0 1; do python -c "
import json;d=json.loads(open('$O/bench_atm$a.json').read().strip().splitlines()[-1]);print('atm$a',d['value'],d['ms_per_step'],[(k,v['us']) for k,v in d['kernel_shares'].items() if 'update' in k])"; done
