# Prefetch at large T (stream) and depth/margin defaults.
set -x
O=gpurun_out/r2o
mkdir -p $O
timeout 300 python tools/trace_timeline.py --scenario t512,t128 --reps 1 > $O/tl_pf.log 2>&1
SNN_LIF_PREFETCH=0 timeout 300 python tools/trace_timeline.py --scenario t512,t128 --reps 1 > $O/tl_nopf.log 2>&1
SNN_LIF_CLC_DEPTH=1 timeout 300 python tools/trace_timeline.py --scenario cfg2,t8 --reps 1 > $O/tl_d1.log 2>&1
for e in "SNN_LIF_PREFETCH=0" "SNN_LIF_PREFETCH=1000" "SNN_LIF_PREFETCH=1000 SNN_LIF_CLC_DEPTH=1"; do
  n=$(echo $e | tr ' =' '__')
  env $e timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/default_$n.json 2> $O/default_$n.err
done
for e in "SNN_LIF_CLC_DEPTH=1 SNN_LIF_CLC_MARGIN=0" "SNN_LIF_CLC_DEPTH=1 SNN_LIF_CLC_MARGIN=2" "SNN_LIF_CLC_DEPTH=1 SNN_LIF_PREFETCH=0" "SNN_LIF_CLC_DEPTH=1"; do
  n=$(echo $e | tr ' =' '__')
  env $e timeout 300 python bench.py --workload cfg2 --no-e2e --no-cpu-baseline > $O/cfg2_$n.json 2> $O/cfg2_$n.err
done
ls -la $O
