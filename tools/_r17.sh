for u in 2 3 4 5 8; do echo "U=$u"; SPB_SPMM_U=$u python tools/bench_spmm.py --config c3 --ld 336 2>/dev/null; SPB_SPMM_U=$u python tools/bench_spmm.py --config c4 --ld 528 2>/dev/null; done
