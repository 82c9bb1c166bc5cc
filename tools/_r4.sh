set -x
O=gpurun_out/r4; mkdir -p $O
python -m pytest tests/test_gpu_update.py tests/test_gpu_gram.py tests/test_gpu_large.py -q -s -p no:cacheprovider -k "not c4" > $O/tests.log 2>&1
for h in 0 0.3 0.5 0.6 0.7 0.8 1.0; do SPB_SPMM_HINT=$h python tools/bench_spmm.py --config c3 --ld 336 >> $O/spmm_hint.log 2>&1; echo "hint=$h" >> $O/spmm_hint.log; done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
SPB_SPMM_HINT=0.6 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3_hint.json 2> $O/bench_c3_hint.err
tail -3 $O/tests.log; cat $O/spmm_hint.log
