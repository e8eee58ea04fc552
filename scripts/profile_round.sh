#!/bin/bash
# ncu evidence for profiles/ (run under gpurun, one GPU):
#   1. launch list of the bench command (per-launch device time)
#   2. --set full captures of the top kernels
set -x
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench.csv \
    python bench.py --steps 3 --warmup 1 --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gate1 -s 3 -c 2 -o $OUT/full_ry30 -f \
    python scripts/prof_targets.py gates 30 > $OUT/full_ry30.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_h2 -c 1 -o $OUT/full_pes -f \
    python scripts/prof_targets.py pes > $OUT/full_pes.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_expect -c 4 -o $OUT/full_expect28 -f \
    python scripts/prof_targets.py expect 28 > $OUT/full_expect28.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_expect_tile -c 2 -o $OUT/full_exptile28f32 -f \
    python scripts/prof_targets.py expect 28 f32 > $OUT/full_exptile28f32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 2 -c 3 -o $OUT/full_tile26 -f \
    python scripts/prof_targets.py hea 26 > $OUT/full_tile26.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 1 -c 2 -o $OUT/full_tile28f32 -f \
    python scripts/prof_targets.py hea 28 f32 > $OUT/full_tile28f32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_vqe_block -c 1 -o $OUT/full_block12 -f \
    python scripts/block_probe.py 12 > $OUT/full_block12.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/block_launches.csv \
    python scripts/block_probe.py 4 8 12 13 > /dev/null 2>&1
ls -la $OUT
