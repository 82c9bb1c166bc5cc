# Bench lines for the round's profiles: C3 (headline) + reference arm, C2, C4.
#   bash tools/round_bench.sh TAG   -> gpurun_out/TAG/bench_*.json
O=gpurun_out/${1:-bench}; mkdir -p $O
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_c3_reference.json 2> $O/bench_c3_reference.err
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
python - "$O" <<'P'
import json, sys
O = sys.argv[1]
for c in ("c3", "c3_reference", "c2", "c4"):
    try:
        d = json.load(open(f"{O}/bench_{c}.json"))
    except Exception as e:
        print(c, "ERR", e); continue
    r = d.get("roofline", {})
    print(c, d.get("ms_per_step"), d.get("value"), d.get("e2e", {}).get("value"), r.get("frac"),
          d.get("step_ms"), d.get("clocks"))
P
