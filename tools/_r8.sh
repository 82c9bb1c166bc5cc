set -x
O=gpurun_out/r8; mkdir -p $O
python -m pytest tests/test_gpu_kmeans.py tests/test_gpu_graph.py tests/test_gpu_lobpcg.py tests/test_gpu_sharded.py -q -s -p no:cacheprovider > $O/tests.log 2>&1
python tools/bench_kmeans.py > $O/kmeans.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
cat $O/kmeans.log; tail -3 $O/tests.log; python -c "
import json;d=json.loads(open('$O/bench_c3.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e'],d['e2e_partition_seconds'])"
