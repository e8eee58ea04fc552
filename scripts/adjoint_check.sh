# GPU check of the adjoint gradient: parity tests, then the scaling study timings (config 3)
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "adjoint or scaling or vqe or fused" > $OUT/pytest_adj.log 2>&1; echo "rc=$?" >> $OUT/pytest_adj.log
timeout 900 python scripts/bench_scaling.py --ref-max 8 --gpu-max 26 > $OUT/scaling2.jsonl 2>&1
