# Round profile set (run on the GPU box): bench lines, launch list, ncu captures.
set -x
O=gpurun_out/prof; mkdir -p $O
timeout 400 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c3 --steps 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c4 --steps 2 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_c2_reference.json 2> $O/bench_c2_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tridiag_warpcol|gram_dmma|chol_wsync|spmm_vb|update_tc" -c 5 -o $O/c2_top python tools/ncu_target.py c2 > $O/ncu_full.log 2>&1
ls -la $O
