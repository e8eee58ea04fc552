L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/ab_keep.so
for i in 1 2; do
  for v in base g3s2 g2s3 r4g4; do
    cp _variants/$v.so $L
    TAG=$v DTYPE=f32 LAYERS=1 timeout 200 python scripts/tile_ab.py 28 30
    TAG=$v DTYPE=f64 LAYERS=1 timeout 200 python scripts/tile_ab.py 30
  done
done
cp /tmp/ab_keep.so $L
