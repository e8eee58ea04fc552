#!/bin/bash
# Full GPU evidence run (gpurun, one B200): tests, smoke, bench (both arms),
# bandwidth sweeps (config 4), fused-circuit timing, scaling study (config 3,
# incl. the shared-memory engine's widths), distributed-state virtual ranks,
# then the ncu captures of scripts/profile_round.sh; with TAG=<round tag> the
# reports are distilled on the box (summary json, per-line stall table).
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.log 2>&1
timeout 600 python bench.py --impl reference > $OUT/bench_ref.log 2>&1
timeout 900 python scripts/bw_sweep.py 26 28 30 32 33 > $OUT/bw_f64.jsonl 2>&1
timeout 900 python scripts/bw_sweep.py 30 32 34 --f32 > $OUT/bw_f32.jsonl 2>&1
timeout 600 python scripts/fusion_check.py > $OUT/fusion_check.log 2>&1
timeout 900 python scripts/mid_width_probe.py 4 5 6 8 10 12 13 14 16 > $OUT/mid_width.jsonl 2>&1
timeout 1500 python scripts/bench_scaling.py --ref-max 16 --gpu-max 26 > $OUT/scaling.jsonl 2>&1
timeout 300 python scripts/dsv_bench.py 30 8 > $OUT/dsv_bench.json 2>&1
if [ "${PROFILE:-1}" = 1 ]; then timeout 2400 bash scripts/profile_round.sh > $OUT/profile.log 2>&1; fi
# distil the ncu reports on the box (gpurun copies back <= 64 MiB): key
# metrics, per-line source exports, then drop the reports
if [ -n "$TAG" ]; then
  python scripts/summarize_ncu.py $TAG > $OUT/summarize.log 2>&1; cp profiles/${TAG}_ncu_summary.json $OUT/ 2>/dev/null
  mkdir -p $OUT/reps
  for f in $OUT/*.ncu-rep; do
    ncu -i $f --page source --csv --print-source cuda,sass --launch-count 1 > $OUT/reps/$(basename $f .ncu-rep)_src.csv 2>/dev/null
  done
  python scripts/stall_lines.py $OUT/reps/*_src.csv > $OUT/${TAG}_stall_lines.txt 2>&1
  rm -f $OUT/*.ncu-rep
fi
echo done
