O=gpurun_out/r15; mkdir -p $O
python tools/ncu_target.py c3 1 > $O/plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:update_tc_kernel -s 21 -c 1 -o $O/ut python tools/ncu_target.py c3 1 > $O/ncu.log 2>&1
ls $O
