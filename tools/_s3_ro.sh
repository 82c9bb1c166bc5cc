O=gpurun_out/ro2; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_reorder.py -x -q -p no:cacheprovider > $O/t_reorder.log 2>&1; tail -15 $O/t_reorder.log
timeout 600 python tools/bench_reorder.py --config c3 > $O/c3.log 2>&1; grep -v Warn $O/c3.log | grep -v sparse_csr
timeout 900 python -m pytest tests/test_gpu_large.py -x -q -s -p no:cacheprovider > $O/t_large.log 2>&1; grep -E 'C3|C4|passed|failed|Error' $O/t_large.log | head -20
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; head -c 400 $O/bench.json; tail -3 $O/bench.err
