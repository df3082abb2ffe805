# Round-2c re-entry check on the restored tree: GPU suite, smoke, default bench line.
O=gpurun_out/r2c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 400 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 400 python bench.py --sweep --no-cpu-baseline --no-e2e > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
ls -la $O
