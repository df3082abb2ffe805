# Final-phase run-ahead A/B (SNN_LIF_RUNAHEAD_MB = 0 / 24 / 48 / 96).
set -x
O=gpurun_out/r2y
mkdir -p $O
for mb in 0 48 96 24; do
  SNN_LIF_RUNAHEAD_MB=$mb timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/default_$mb.json 2> $O/default_$mb.err
  SNN_LIF_RUNAHEAD_MB=$mb timeout 300 python bench.py --sweep --no-e2e --no-cpu-baseline > $O/sweep_$mb.json 2> $O/sweep_$mb.err
done
SNN_LIF_RUNAHEAD_MB=0 timeout 300 python bench.py --workload cfg4 --no-e2e --no-cpu-baseline > $O/cfg4_0.json 2> $O/cfg4_0.err
SNN_LIF_RUNAHEAD_MB=48 timeout 300 python bench.py --workload cfg4 --no-e2e --no-cpu-baseline > $O/cfg4_48.json 2> $O/cfg4_48.err
SNN_LIF_RUNAHEAD_MB=48 timeout 300 python tools/trace_timeline.py --scenario t512,t128 --reps 1 > $O/tl_48.log 2>&1
SNN_LIF_RUNAHEAD_MB=0 timeout 300 python tools/trace_timeline.py --scenario t512,t128 --reps 1 > $O/tl_0.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
ls -la $O
