set -x
O=gpurun_out/r9; mkdir -p $O
python -m pytest tests/test_gpu_graph.py tests/test_gpu_sharded.py tests/test_gpu_large.py -q -s -p no:cacheprovider -k "graph or bit_exact or sharded or hub or symmetrize or c3_partition" > $O/tests.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config c4 > $O/bench_c4.json 2> $O/bench_c4.err
tail -3 $O/tests.log; grep -n "FAILED" $O/tests.log | head; for c in c3 c4; do python -c "
import json;d=json.loads(open('$O/bench_$c.json').read().strip().splitlines()[-1]);print('$c',d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['csr_build']['ms_per_build'],d['roofline']['csr_build']['achieved'],d['quality'])"; done
