# New scheduling defaults (depth 1, short-tile prefetch) vs a 512/256-neuron tile variant.
set -x
O=gpurun_out/r2p
mkdir -p $O
W=paper_2408_00280_b200/build_w512/libsnn_lif_w512.so
for v in base w512; do
  if [ $v = w512 ]; then export SNN_LIF_LIBRARY=$W; else unset SNN_LIF_LIBRARY; fi
  timeout 300 python bench.py --workload cfg2 --no-e2e --no-cpu-baseline > $O/cfg2_$v.json 2> $O/cfg2_$v.err
  timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/default_$v.json 2> $O/default_$v.err
  timeout 300 python bench.py --workload cfg4 --no-e2e --no-cpu-baseline > $O/cfg4_$v.json 2> $O/cfg4_$v.err
  timeout 300 python bench.py --sweep --no-e2e --no-cpu-baseline > $O/sweep_$v.json 2> $O/sweep_$v.err
done
unset SNN_LIF_LIBRARY
timeout 300 python tools/trace_timeline.py --scenario cfg2,t512 --reps 1 > $O/tl_base.log 2>&1
ls -la $O
