# GPU check of the fused tile path: parity tests, then fused vs per-gate timing (scripts/fusion_check.py)
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_tile.log 2>&1; echo "rc=$?" >> $OUT/pytest_tile.log
timeout 600 python scripts/fusion_check.py > $OUT/fusion_check.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 2 -c 3 -o $OUT/full_tile26 python scripts/prof_targets.py hea 26 > $OUT/full_tile26.log 2>&1
