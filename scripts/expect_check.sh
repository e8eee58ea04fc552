# GPU check of the expectation kernels: parity tests, bandwidth at n = 28/30, ncu capture of the multi-group pass
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "expectation or adjoint or scaling or tfim" > $OUT/pytest_expect.log 2>&1; echo "rc=$?" >> $OUT/pytest_expect.log
timeout 600 python scripts/bw_sweep.py 28 30 > $OUT/bw_28_30.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_expect_multi -c 3 -o $OUT/full_expect28 python scripts/prof_targets.py expect 28 > $OUT/full_expect28.log 2>&1
