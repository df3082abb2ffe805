# 3-D block tensor maps (one TMA load per tensor per stage): GPU suite + A/B SNN_LIF_BLK3=0/1.
set -x
O=gpurun_out/r2ac
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for b in 0 1; do
  SNN_LIF_BLK3=$b timeout 300 python bench.py --workload cfg2 --no-e2e --no-cpu-baseline > $O/cfg2_$b.json 2> $O/cfg2_$b.err
  SNN_LIF_BLK3=$b timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/default_$b.json 2> $O/default_$b.err
  SNN_LIF_BLK3=$b timeout 300 python bench.py --sweep --no-e2e --no-cpu-baseline > $O/sweep_$b.json 2> $O/sweep_$b.err
  SNN_LIF_BLK3=$b timeout 300 python bench.py --workload cfg4 --no-e2e --no-cpu-baseline > $O/cfg4_$b.json 2> $O/cfg4_$b.err
  SNN_LIF_BLK3=$b timeout 300 python tools/trace_timeline.py --scenario cfg2 --reps 1 > $O/tl_$b.log 2>&1
done
ls -la $O
