#!/bin/bash
# A/B of environment settings on c4 (or $CFG): one bench line per setting.
#   scripts/ab_env.sh "" "FHT_TILE_WIDTH=32 FHT_K2_SMEM_KB=125"
CFG=${CFG:-c4}
mkdir -p gpurun_out/ab
i=0
for e in "$@"; do
  env $e python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab/$i.json 2> gpurun_out/ab/$i.err
  python - "$i" "$e" <<'PY'
import json, sys
try:
    d = json.load(open(f"gpurun_out/ab/{sys.argv[1]}.json"))
    r = d["roofline"]
    print(f"[{sys.argv[2]}] {d['value']:.1f} Gsums/s {d['ms_per_step']:.4f} ms", {k: round(v, 4) for k, v in r["kernel_ms"].items()})
except Exception as ex:
    print(f"[{sys.argv[2]}] failed: {ex}", open(f"gpurun_out/ab/{sys.argv[1]}.err").read()[-800:])
PY
  i=$((i+1))
done
