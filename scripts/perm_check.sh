L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/keep.so
for v in s4 s6; do cp _variants/$v.so $L; echo "== $v"; timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k large_register 2>&1 | tail -1; done
cp /tmp/keep.so $L
