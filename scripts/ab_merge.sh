# A/B: TMA run merging in k_tile (VQF_TILE_NO_MERGE=1 disables it)
for i in 1 2; do
  for m in 0 1; do
    for dt in f32 f64; do
      if [ $m = 1 ]; then export VQF_TILE_NO_MERGE=1; else unset VQF_TILE_NO_MERGE; fi
      TAG=nomerge$m DTYPE=$dt LAYERS=1 timeout 200 python scripts/tile_ab.py 28 30
    done
  done
done
