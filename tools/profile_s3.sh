# Round-2 (session 3) profile set at C3/C4 with the SpMM locality order: launch list
# and full ncu captures of the top kernels. Outputs in gpurun_out/s3prof/.
O=gpurun_out/s3prof; mkdir -p $O
python tools/ncu_target.py c3 1 > $O/target_c3.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_c3.csv python tools/ncu_target.py c3 1 > $O/ncu_launch.log 2>&1
for spec in "spmm_vb 5 1" "update_tc_kernel 20 6" "gram_oz_kernel 10 2" "oz_pack 10 1"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$1 -s $2 -c $3 -o $O/c3_$1 python tools/ncu_target.py c3 1 > $O/ncu_$1.log 2>&1
done
python tools/ncu_target.py c4 1 > $O/target_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:spmm_vb -s 3 -c 1 -o $O/c4_spmm_vb python tools/ncu_target.py c4 1 > $O/ncu_c4_spmm.log 2>&1
ls -la $O
