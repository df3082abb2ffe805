# Prefetch policy A/B (no hint vs evict-first hint; always vs short tiles only) on the stream sweep and cfg2.
set -x
O=gpurun_out/r2q
mkdir -p $O
for e in "SNN_LIF_PREFETCH=0" "SNN_LIF_PREFETCH=1000" "SNN_LIF_PREFETCH=1000 SNN_LIF_PREFETCH_HINT=1" "SNN_LIF_PREFETCH=4"; do
  n=$(echo $e | tr ' =' '__')
  env $e timeout 300 python bench.py --sweep --no-e2e --no-cpu-baseline > $O/sweep_$n.json 2> $O/sweep_$n.err
  env $e timeout 300 python bench.py --workload cfg2 --no-e2e --no-cpu-baseline > $O/cfg2_$n.json 2> $O/cfg2_$n.err
done
SNN_LIF_PREFETCH=1000 SNN_LIF_PREFETCH_HINT=1 timeout 300 python tools/trace_timeline.py --scenario t512,t8 --reps 1 > $O/tl_hint.log 2>&1
ls -la $O
