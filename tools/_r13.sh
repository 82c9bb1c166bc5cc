set -x
O=gpurun_out/r13; mkdir -p $O
python -m pytest tests -m gpu -q -s -p no:cacheprovider > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
python bench.py --steps 20 --warmup 5 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --steps 20 --warmup 5 --config c2 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
python tools/e2e_profile.py --config c3 > $O/e2e_c3.log 2>&1
tail -3 $O/gputest.log; grep -n "FAILED" $O/gputest.log | head
