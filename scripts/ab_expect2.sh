# A/B of expectation-pass builds (VARIANTS, _variants/<name>.so) vs the current
# build, TFIM at n = 28 / 30 in fp64 and fp32, plus the current build with the
# fp32 diagonal fold forced on (VQF_DIAG_FOLD32=1)
L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/new.so
for i in 1 2; do
 for v in ${VARIANTS:-expold} new; do
  if [ $v = new ]; then cp /tmp/new.so $L; else cp _variants/$v.so $L; fi
  for dt in f64 f32; do TAG=$v DTYPE=$dt timeout 200 python scripts/expect_ab.py 28 30; done
 done
 TAG=new-fold32 DTYPE=f32 VQF_DIAG_FOLD32=1 timeout 200 python scripts/expect_ab.py 28 30
done
cp /tmp/new.so $L
