# r2c: checkpoint row 0 elided -- GPU suite, smoke, small-T probe, cfg2 / default bench lines.
O=gpurun_out/r2c_ck0; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -rs > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 300 python tools/small_t_probe.py --T 8,16,32,128 --preps clean,dirty --families tma > $O/small_t_probe.log 2>&1
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 400 python bench.py --no-cpu-baseline --no-e2e > $O/bench_default.json 2> $O/bench_default.err
