# A/B of fused-tile builds: _variants/<name>.so (VARIANTS) vs the current build, one HEA layer, fp32 + fp64
L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/new.so
for i in 1 2; do
 for v in ${VARIANTS:-tunf} new; do
  if [ $v = new ]; then cp /tmp/new.so $L; else cp _variants/$v.so $L; fi
  for dt in f32 f64; do TAG=$v DTYPE=$dt LAYERS=1 timeout 200 python scripts/tile_ab.py 28 30; done
 done
done
cp /tmp/new.so $L
