# A/B of the unaligned-row consumer changes (funnel-shift spike stores, widest smem loads).
set -x
O=gpurun_out/r2v
mkdir -p $O
for v in base noshift elemlds both; do
  if [ $v = base ]; then unset SNN_LIF_LIBRARY; else export SNN_LIF_LIBRARY=paper_2408_00280_b200/build_$v/libsnn_lif_$v.so; fi
  timeout 300 python tools/kbench.py --cases unal > $O/kbench_$v.log 2>&1
done
ls -la $O
