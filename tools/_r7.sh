set -x
O=gpurun_out/r7; mkdir -p $O
python tools/h2d_bench.py > $O/h2d.log 2>&1
python -m pytest tests/test_gpu_kmeans.py tests/test_gpu_gram.py -q -s -p no:cacheprovider > $O/tests.log 2>&1
python tools/bench_kmeans.py > $O/kmeans.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
cat $O/h2d.log $O/kmeans.log; tail -5 $O/tests.log; tail -2 $O/smoke.log
