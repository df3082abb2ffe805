# Round-2 second GPU pass: the NCCL C-ABI time split (1 rank and 2 ranks on one GPU), the bench
# multi-rank paths, the full GPU suite, default bench line.
set -x
O=gpurun_out/r2b
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_comm.py -x -q -p no:cacheprovider -rs > $O/pytest_comm.log 2>&1; echo "rc=$?" >> $O/pytest_comm.log
timeout 900 python -m pytest tests/test_gpu_bench.py -x -q -p no:cacheprovider -rs > $O/pytest_bench.log 2>&1; echo "rc=$?" >> $O/pytest_bench.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 400 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 400 python bench.py --workload cfg3 --steps 5 --no-e2e > $O/bench_cfg3_k1.json 2> $O/bench_cfg3_k1.err
ls -la $O
