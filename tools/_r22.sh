for e in 0 1 2 4 3 5 6 7; do echo "EXP=$e"; SPB_UT_EXP=$e python tools/bench_update.py --shapes 500000x324x108,500000x108x108 2>&1 | tail -2; done
