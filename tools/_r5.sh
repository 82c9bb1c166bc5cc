set -x
O=gpurun_out/r5; mkdir -p $O
python -m pytest tests/test_gpu_update.py tests/test_gpu_gram.py tests/test_gpu_large.py -q -s -p no:cacheprovider -k "not c4" > $O/tests.log 2>&1
for cfg in "0 0" "56 0" "56 1.0" "36 1.0" "28 1.0" "56 0.6"; do set -- $cfg; SPB_SPMM_PANEL=$1 SPB_SPMM_HINT=$2 python tools/bench_spmm.py --config c3 --ld 336 2>/dev/null >> $O/spmm_panel.log; echo "panel=$1 hint=$2" >> $O/spmm_panel.log; done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
grep -n "C3 \|C5 \|passed\|failed" $O/tests.log; cat $O/spmm_panel.log
