O=gpurun_out/chk2; mkdir -p $O
python tools/ab_step.py --steps 6 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_update.py tests/test_gpu_gram.py tests/test_gpu_kmeans.py tests/test_gpu_large.py -x -q -s -p no:cacheprovider > $O/t.log 2>&1; grep -E 'C3|C4|passed|failed|Error' $O/t.log | head -20
