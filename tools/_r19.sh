O=gpurun_out/r19; mkdir -p $O
python -m pytest tests/test_gpu_lobpcg.py tests/test_gpu_large.py -q -p no:cacheprovider -k "not c4 and not c5" > $O/tests.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
tail -2 $O/tests.log; python -c "
import json;d=json.loads(open('$O/bench_c3.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e'],d['e2e_partition_seconds'])"
