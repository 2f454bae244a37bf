set -u
CFGS=${CFGS:-"c4 c5 c3 c2 c1"}
for c in $CFGS; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline $EXTRA > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo $c rc $?; tail -2 gpurun_out/b_$c.err; done
python - <<PY
import json
for c in "$CFGS".split():
    try:
        d=json.load(open(f"gpurun_out/b_{c}.json"))
        r=d["roofline"]
        print(c, "val", d["value"], "ms", d["ms_per_step"], r["kernel"], "frac", r["frac"], r["kernel_ms"], r.get("kernel_gbs"), "stepGBs", d["hbm_gbs_step"], "e2e", (d["e2e"] or {}).get("value"))
    except Exception as e: print(c, "ERR", e)
PY
