#!/bin/bash
# One GPU session: tests, smoke, bench, then ncu evidence (scripts/profile_round.sh).
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 600 python bench.py --impl reference > $OUT/bench_ref.log 2>&1
if [ "${PROFILE:-1}" = 1 ]; then timeout 1500 bash scripts/profile_round.sh > $OUT/profile.log 2>&1; fi
tail -3 $OUT/pytest_gpu.log $OUT/smoke.log $OUT/bench.log $OUT/bench_ref.log
