for i in 1 2; do for dt in f64 f32; do
  TAG=fold DTYPE=$dt python scripts/expect_ab.py 28 30
  VQF_NO_DIAG_FOLD=1 TAG=nofold DTYPE=$dt python scripts/expect_ab.py 28 30
done; done
