# compute-sanitizer over the affine / residual prologue kernels + the new GPU tests.
mkdir -p gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck racecheck; do
  echo "== $tool"; timeout 600 $CS --tool $tool --print-limit 20 python tools/san_affine.py 2>&1 | tail -8
done
timeout 600 python -m pytest -m gpu -x -q tests/test_gpu_parity.py -k "residual" 2>&1 | tail -3
