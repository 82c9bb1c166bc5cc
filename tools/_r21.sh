O=gpurun_out/r21; mkdir -p $O
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/c3.json 2> $O/c3.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config c2 > $O/c2.json 2> $O/c2.err
for c in c3 c2; do python -c "
import json;d=json.loads(open('$O/'+'$c'+'.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$c',d['value'],{k:r[k] for k in ('bound','achieved','peak','unit','frac','launches','avg_launch_us','live_ms_total')}, r.get('spmm',r.get('gram',{})).get('frac'))"; done
