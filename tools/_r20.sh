O=gpurun_out/r20; mkdir -p $O
SPB_SHARD_TRANSPORT=host timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 > $O/bench_n2.json 2> $O/bench_n2.err
echo "rc=$?"; tail -c 1500 $O/bench_n2.json; tail -5 $O/bench_n2.err
