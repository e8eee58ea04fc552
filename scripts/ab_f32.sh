# fp32 k_tile shape A/B (scripts/build_variant.sh variants)
L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/keep.so
for i in 1 2; do for v in "$@"; do cp _variants/$v.so $L; TAG=$v DTYPE=f32 LAYERS=1 timeout 200 python scripts/tile_ab.py 28 30; done; done
cp /tmp/keep.so $L
