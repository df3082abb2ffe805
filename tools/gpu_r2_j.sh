set -x
O=gpurun_out/r2j
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench.py tests/test_gpu_comm.py -q -p no:cacheprovider -rs -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 400 python bench.py --sweep --no-cpu-baseline --no-e2e --steps 5 > $O/bench_sweep.json 2> $O/bench_sweep.err
