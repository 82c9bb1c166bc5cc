O=gpurun_out/s3base; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider -s > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -3 $O/gputest.log; cat $O/bench.json | head -c 600
