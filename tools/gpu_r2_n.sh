# A/B of the launch scheduling knobs (early L2 prefetch, CLC hoarding margin, depth) on cfg2 and the cfg1 sweep.
set -x
O=gpurun_out/r2n
mkdir -p $O
ab() {   # name, env...
  n=$1; shift
  env "$@" timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/cfg2_$n.json 2> $O/cfg2_$n.err
  env "$@" timeout 300 python bench.py --sweep --no-cpu-baseline --no-e2e > $O/sweep_$n.json 2> $O/sweep_$n.err
}
ab old SNN_LIF_PREFETCH=0 SNN_LIF_CLC_MARGIN=0
ab pf SNN_LIF_CLC_MARGIN=0
ab m1 SNN_LIF_PREFETCH=0 SNN_LIF_CLC_MARGIN=1
ab pf_m1 SNN_LIF_CLC_MARGIN=1
ab pf_m2 SNN_LIF_CLC_MARGIN=2
ab pf_d2 SNN_LIF_CLC_DEPTH=2 SNN_LIF_CLC_MARGIN=0
ab pf_d1 SNN_LIF_CLC_DEPTH=1
timeout 300 python tools/trace_timeline.py --scenario cfg2,t8,t32 --reps 1 > $O/timeline_new.log 2>&1
SNN_LIF_PREFETCH=0 SNN_LIF_CLC_MARGIN=0 timeout 300 python tools/trace_timeline.py --scenario cfg2 --reps 1 > $O/timeline_old.log 2>&1
timeout 400 python bench.py --no-e2e --no-cpu-baseline > $O/default.json 2> $O/default.err
ls -la $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
