# k_tile ring sizes (scripts/build_variant.sh s4 / s6): fused vs per-gate
# results and one HEA layer's time for each
L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/keep.so
for v in s4 s6; do
  cp _variants/$v.so $L
  TAG=$v python scripts/ring_probe.py 16 20 24 28 2>&1 | grep n=
  for dt in f64 f32; do TAG=$v DTYPE=$dt LAYERS=1 python scripts/tile_ab.py 28 30 2>&1 | grep n=; done
done
cp /tmp/keep.so $L
