O=gpurun_out/r12; mkdir -p $O
python tools/csr_target.py c3 2 > $O/plain.log 2>&1; python tools/csr_target.py c4 2 >> $O/plain.log 2>&1
python -m pytest tests/test_gpu_graph.py -q -p no:cacheprovider > $O/tests.log 2>&1
python tools/csr_target.py c3 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/csr_launches.csv python tools/csr_target.py c3 1 > $O/ncu.log 2>&1
cat $O/plain.log; tail -2 $O/tests.log; python tools/ncu_summary.py $O/csr_launches.csv "csr c3" | head -12
