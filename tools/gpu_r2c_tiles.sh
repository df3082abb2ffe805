# fp32 forward tile-geometry A/B at small T (clean flush), default vs variant builds.
O=gpurun_out/r2c; mkdir -p $O
for v in default w512 w256; do
  if [ $v = default ]; then L=""; else L=paper_2408_00280_b200/build_$v/libsnn_lif_$v.so; fi
  echo "== $v" >> $O/tiles.log
  SNN_LIF_LIBRARY=$L timeout 300 python tools/small_t_probe.py --T 8,16,32,128,512 --preps clean --families tma >> $O/tiles.log 2>&1
done
