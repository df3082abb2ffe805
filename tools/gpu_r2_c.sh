# Round-2 third GPU pass: the unaligned-row TMA kernels -- GPU suite, sanitizers, kbench A/B.
set -x
O=gpurun_out/r2c
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rs -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/kbench.py --cases unal,sweep,cfg2 > $O/kbench.log 2>&1
for tool in memcheck synccheck initcheck; do
  echo "== $tool" >> $O/san.log; timeout 900 $CS --tool $tool --print-limit 20 python tools/san_unaligned.py >> $O/san.log 2>&1; echo "rc=$?" >> $O/san.log
done
timeout 400 python bench.py --no-cpu-baseline > $O/bench_default.json 2> $O/bench_default.err
ls -la $O
