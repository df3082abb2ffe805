set -x
O=gpurun_out/r2f
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_plan.py -m gpu -q -p no:cacheprovider -x -k "affine or plan" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --T 32 --no-e2e --no-cpu-baseline --affine --prologue > $O/bench_affine.json 2> $O/bench_affine.err
