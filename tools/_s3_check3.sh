O=gpurun_out/chk3; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_update.py tests/test_gpu_kmeans.py -x -q -p no:cacheprovider > $O/t0.log 2>&1; tail -3 $O/t0.log
python tools/ab_step.py --steps 6 2>&1 | tail -1
python tools/ab_step.py --steps 2 --config c4 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_lobpcg.py -x -q -s -p no:cacheprovider > $O/t.log 2>&1; grep -E 'C3|C4|passed|failed|Error' $O/t.log | head -20
