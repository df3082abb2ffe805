# Ring depth A/B: fp32 forward/backward with 2 stages instead of 3 (fewer bytes in flight).
set -x
O=gpurun_out/r2z
mkdir -p $O
for v in base s2; do
  if [ $v = base ]; then unset SNN_LIF_LIBRARY; else export SNN_LIF_LIBRARY=paper_2408_00280_b200/build_$v/libsnn_lif_$v.so; fi
  timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/default_$v.json 2> $O/default_$v.err
  timeout 300 python tools/kbench.py --cases cfg1,sweep > $O/kbench_$v.log 2>&1
done
ls -la $O
