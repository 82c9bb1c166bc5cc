# Launch list of one C3 partition (ncu, gpu__time_duration only) into gpurun_out/$1/.
O=gpurun_out/${1:-launches}; mkdir -p $O
python tools/ncu_target.py c3 1 > $O/target_c3.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_c3.csv python tools/ncu_target.py c3 1 > $O/ncu_launch.log 2>&1
