# Fused-layer timing of the current build (fp32 and fp64, one HEA layer)
for i in 1 2; do for dt in f32 f64; do TAG=cur DTYPE=$dt LAYERS=1 timeout 200 python scripts/tile_ab.py 28 30; done; done
