# A/B of expectation-pass builds: _variants/<name>.so vs the current build
L=paper_2601_09951_b200/libvqf_b200.so
cp $L /tmp/new.so
for i in 1 2; do
 for v in ${VARIANTS:-expold} new; do
  if [ $v = new ]; then cp /tmp/new.so $L; else cp _variants/$v.so $L; fi
  for dt in f64 f32; do TAG=$v DTYPE=$dt timeout 200 python scripts/expect_ab.py 28 30; done
 done
done
cp /tmp/new.so $L
