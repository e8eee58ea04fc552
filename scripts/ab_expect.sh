# Expectation A/B of library builds under _variants/: bash scripts/ab_expect.sh base tree
L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/ab_keep.so
for i in 1 2; do for v in "$@"; do cp _variants/$v.so $L; TAG=$v timeout 200 python scripts/expect_ab.py 28 30; done; done
cp /tmp/ab_keep.so $L
