# r2c: unaligned u8x4 spike-store A/B (0: predicated .cs [product], 1: four byte stores, 2: predicated plain).
O=gpurun_out/r2c_u8ab; mkdir -p $O
for v in default u8m1 u8m2; do
  if [ $v = default ]; then L=""; else L=paper_2408_00280_b200/build_$v/libsnn_lif_$v.so; fi
  echo "== $v" >> $O/kbench.log
  SNN_LIF_LIBRARY=$L timeout 300 python tools/kbench.py --cases unal --reps 20 >> $O/kbench.log 2>&1
done
