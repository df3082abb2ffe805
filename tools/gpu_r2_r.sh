# Half-width tail tiles: correctness (GPU suite) and A/B (SNN_LIF_SPLIT_TAIL=0/1).
set -x
O=gpurun_out/r2r
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for e in "SNN_LIF_SPLIT_TAIL=0" "SNN_LIF_SPLIT_TAIL=1"; do
  n=$(echo $e | tr ' =' '__')
  env $e timeout 300 python bench.py --workload cfg2 --no-e2e --no-cpu-baseline > $O/cfg2_$n.json 2> $O/cfg2_$n.err
  env $e timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/default_$n.json 2> $O/default_$n.err
  env $e timeout 300 python bench.py --workload cfg4 --no-e2e --no-cpu-baseline > $O/cfg4_$n.json 2> $O/cfg4_$n.err
  env $e timeout 300 python bench.py --sweep --no-e2e --no-cpu-baseline > $O/sweep_$n.json 2> $O/sweep_$n.err
  env $e timeout 300 python tools/trace_timeline.py --scenario cfg2,t512,t8 --reps 1 > $O/tl_$n.log 2>&1
done
ls -la $O
