# Round-2 re-entry check: the committed tree on a fresh box (GPU suite, default bench line, per-kernel small-shape timings).
set -x
O=gpurun_out/r2l
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 400 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python tools/kbench.py --cases sweep,cfg2,small,unal > $O/kbench.log 2>&1
ls -la $O
