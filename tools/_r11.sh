O=gpurun_out/r11; mkdir -p $O
python tools/csr_target.py c3 1 > $O/plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:bk_rows -s 1 -c 1 -o $O/bk_rows python tools/csr_target.py c3 1 > $O/ncu.log 2>&1
ls -la $O
