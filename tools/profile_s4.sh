# Session-4 profile set (C3, plus the C4 SpMM and Gram): launch list and full ncu
# captures of the top kernels. Outputs in gpurun_out/s4final/; summaries go to
# profiles/r02/s4/ (tools/ncu_brief.py, tools/ncu_summary.py).
O=gpurun_out/s4final; mkdir -p $O
python tools/ncu_target.py c3 1 > $O/target_c3.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_c3.csv python tools/ncu_target.py c3 1 > $O/ncu_launch.log 2>&1
for spec in "gram_oz_kernel 10 1" "spmm_vb 5 1" "update_tc_kernel 20 3" "tridiag_cluster_mb 5 1" "oz_pack 10 1" "qrcp_pivots 0 1" "chol_rowwarp 5 1"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$1 -s $2 -c $3 -o $O/c3_$1 python tools/ncu_target.py c3 1 > $O/ncu_$1.log 2>&1
done
python tools/ncu_target.py c4 1 > $O/target_c4.log 2>&1 && \
for spec in "spmm_vb 3 1" "gram_oz_kernel 10 1"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none -k regex:$1 -s $2 -c $3 -o $O/c4_$1 python tools/ncu_target.py c4 1 > $O/ncu_c4_$1.log 2>&1
done
ls -la $O
