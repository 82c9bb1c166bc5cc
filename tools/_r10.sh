O=gpurun_out/r10; mkdir -p $O
python tools/csr_target.py c3 2 > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/csr_launches.csv python tools/csr_target.py c3 1 > $O/ncu.log 2>&1
cat $O/plain.log; python tools/ncu_summary.py $O/csr_launches.csv "csr c3" | head -20
