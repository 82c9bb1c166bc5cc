O=gpurun_out/s3prof2; mkdir -p $O
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err
python - <<'P'
import json; d=json.load(open('gpurun_out/s3prof2/bench.json')); r=d['roofline']
print(d['ms_per_step'], d['value'], d['e2e']['value'], r['kernel'], r['frac'])
for k,v in d['kernel_shares'].items(): print(f"{v['us']:10.1f} {v['launches']:5d} {k}")
P
for spec in "update_tc_kernel 20 3" "gram_oz_kernel 10 1"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$1 -s $2 -c $3 -o $O/c3_$1 python tools/ncu_target.py c3 1 > $O/ncu_$1.log 2>&1
done
python tools/ncu_brief.py $O/c3_update_tc_kernel.ncu-rep $O/c3_gram_oz_kernel.ncu-rep | grep -E '==|duration|tensor|DRAM thr|issue|stall'
