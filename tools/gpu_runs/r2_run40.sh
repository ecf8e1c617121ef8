# K1 variants (ILP x min CTAs/SM) vs the committed kernel: standalone roofline at 8192 and 65536 patches
cp paper_1205_5351_b200/libtilt.so /tmp/libtilt_base.so
for v in base k1_2_4 k1_2_3 k1_4_3; do
  if [ $v = base ]; then cp /tmp/libtilt_base.so paper_1205_5351_b200/libtilt.so; else cp paper_1205_5351_b200/libtilt_$v.so paper_1205_5351_b200/libtilt.so; fi
  for N in 8192 65536; do echo "$v $N $(timeout 300 python tools/k1_run.py $N 2>&1 | tail -1)" | tee -a gpurun_out/r2_k1_variants.log; done
done
