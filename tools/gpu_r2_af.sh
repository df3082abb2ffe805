# 8-row-stage backward for T <= 8: GPU suite + A/B (SNN_LIF_SHORT_BWD=0/1).
set -x
O=gpurun_out/r2af
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for b in 0 1; do
  SNN_LIF_SHORT_BWD=$b timeout 300 python bench.py --sweep --no-e2e --no-cpu-baseline > $O/sweep_$b.json 2> $O/sweep_$b.err
  SNN_LIF_SHORT_BWD=$b timeout 300 python tools/kbench.py --cases sweep > $O/kbench_$b.log 2>&1
done
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 10 python tools/san_ragged.py > $O/san_memcheck.log 2>&1; echo "rc=$?" >> $O/san_memcheck.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 10 python tools/san_ragged.py > $O/san_synccheck.log 2>&1; echo "rc=$?" >> $O/san_synccheck.log
ls -la $O
