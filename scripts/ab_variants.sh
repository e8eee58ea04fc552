# A/B of library builds kept under _variants/ (git-ignored): each variant's
# libvqf_b200.so is copied into place and timed with scripts/tile_ab.py.
#   bash scripts/ab_variants.sh old direct
L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/ab_keep.so
for i in 1 2; do
  for v in "$@"; do
    cp _variants/$v.so $L
    for layers in 1 2; do TAG=$v LAYERS=$layers timeout 200 python scripts/tile_ab.py 26 30; done
  done
done
cp /tmp/ab_keep.so $L
