# A/B/C/... kernel timing across library builds in ab/ (tuning aid).
# usage: bash tools/gpu_ab_multi.sh "<cases>" lib1 lib2 ...
cases=$1; shift
for rep in 1 2; do
  for l in "$@"; do
    echo "== $l ($rep)"; SNN_LIF_LIBRARY=$PWD/ab/$l timeout 300 python tools/kbench.py --cases $cases
  done
done
