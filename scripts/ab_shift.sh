# Parameter-shift latency A/B of library builds under _variants/:
#   bash scripts/ab_shift.sh r01h cur
L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/ab_keep.so
for i in 1 2; do
  for v in "$@"; do
    cp _variants/$v.so $L
    echo "== $v"; timeout 200 python scripts/shift_repeat_probe.py 8 12 20
  done
done
cp /tmp/ab_keep.so $L
