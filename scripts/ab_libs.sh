# A/B of library builds on one box: bash scripts/ab_libs.sh CONFIG ENV lib1.so lib2.so ...
cfg=$1; shift; envs=$1; shift
cp paper_2411_07351_b200/libfht_b200.so /tmp/lib_orig.so
for l in "$@"; do
  cp "$l" paper_2411_07351_b200/libfht_b200.so
  env $envs timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));r=d['roofline'];print('$cfg','$l','$envs',d['value'],d['ms_per_step'],r['kernel_ms'])"
done
cp /tmp/lib_orig.so paper_2411_07351_b200/libfht_b200.so
