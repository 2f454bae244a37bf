#!/bin/bash
# One GPU-box evidence run: benches (c4 default + c1/c2/c3/c5), the reference
# arm, the ncu launch list of the c4 bench command and full captures of the
# c4 and c5 kernels.  Outputs under gpurun_out/ev/.
set -u
O=gpurun_out/ev; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.csv 2>&1
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo "bench c4 rc $?"
for c in c1 c2 c3 c5; do python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc $?"; done
python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference_c4.json 2> $O/bench_reference.err; echo "ref rc $?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k_stage" -c 400 --csv --log-file $O/launches_c4.csv $CMD > $O/ncu_launches.log 2>&1; echo "ncu launches rc $?"
python scripts/profile_case.py --config c4 --iters 2 > $O/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k1_by32|k1_blocks|k2_pass|k2_pair_pipe|k_stage" -s 4 -c 4 -o $O/full_c4 python scripts/profile_case.py --config c4 --iters 2 > $O/ncu_full_c4.log 2>&1; echo "ncu c4 rc $?"
python scripts/profile_case.py --config c5 --iters 2 > $O/plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k1_by32|k2_pass" -s 3 -c 3 -o $O/full_c5 python scripts/profile_case.py --config c5 --iters 2 > $O/ncu_full_c5.log 2>&1; echo "ncu c5 rc $?"
