# A/B of the projected-eigensolve kernels (diagnostics)
exec 2>/dev/null
for m in 49 63 147 324; do timeout 60 python tools/bench_small.py --m $m --gb; SPB_CHOL_ROWWARP=0 timeout 60 python tools/bench_small.py --m $m --gb; done
timeout 400 python -m pytest tests -m gpu -q 2>&1 | tail -3
