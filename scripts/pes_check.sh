# GPU check of the PES engine: parity tests (goldens, tol-mode counts, large theta), bench, stage clocks
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "sweep or vqe or h2 or pes" > $OUT/pytest_pes.log 2>&1; echo "rc=$?" >> $OUT/pytest_pes.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_pes.log 2>&1
timeout 300 bash scripts/stage_clocks.sh > $OUT/stage_clocks.txt 2>&1
