# A/B of k_tile ring sizes (scripts/build_variant.sh s4 / s5 / s6)
L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/ab_keep.so
for i in 1 2; do
  for v in s4 s5 s6; do
    cp _variants/$v.so $L
    for dt in f32 f64; do TAG=$v DTYPE=$dt LAYERS=1 timeout 200 python scripts/tile_ab.py 28 30; done
  done
done
cp /tmp/ab_keep.so $L
