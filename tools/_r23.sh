O=gpurun_out/r23; mkdir -p $O
python -m pytest tests/test_gpu_streaming.py tests/test_gpu_large.py -q -s -p no:cacheprovider -k "stream or c5" > $O/tests.log 2>&1
python tools/bench_stream.py > $O/c5.json 2> $O/c5.err
tail -2 $O/tests.log; grep FAILED $O/tests.log; cat $O/c5.err | tail -4
