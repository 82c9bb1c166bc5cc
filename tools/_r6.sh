set -x
O=gpurun_out/r6; mkdir -p $O
python -m pytest tests -m gpu -q -s -p no:cacheprovider > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
python bench.py --steps 20 --warmup 5 > $O/bench_c3.json 2> $O/bench_c3.err
python tools/bench_stream.py --reference > $O/c5.json 2> $O/c5.err
grep -n "C3 \|C4 \|C5 \|world=\|passed\|failed" $O/gputest.log | tail -40; tail -3 $O/c5.err
