# A/B of environment settings on one box: bash scripts/ab.sh CONFIG "ENV1" "ENV2" ...
cfg=$1; shift
for e in "$@"; do
  env $e timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));r=d['roofline'];print('$cfg','$e',d['value'],d['ms_per_step'],r['kernel_ms'])"
done
