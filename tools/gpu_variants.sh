# Bench-line variants of the default workload (spike format / save mode) for DESIGN.md.
O=gpurun_out/var; mkdir -p $O
for v in "--spike-fmt bits" "--spike-fmt io" "--save-mode h" "--save-mode h --spike-fmt bits"; do
  n=$(echo $v | tr -d ' -'); timeout 300 python bench.py $v --no-cpu-baseline --no-e2e > $O/b_$n.json 2> $O/b_$n.err
done
timeout 300 python bench.py --workload cfg2 --spike-fmt io --no-cpu-baseline --no-e2e > $O/b_cfg2_io.json 2> $O/b_cfg2_io.err
ls -la $O
