for e in "" "FHT_HOST_PARTS=16" "FHT_HOST_PARTS=32" "FHT_HOST_PARTS=4"; do
  env $e python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e2e.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e2e.json'));print('[$e]', d['e2e']['value'], d['e2e']['ms_per_step'])"
done
