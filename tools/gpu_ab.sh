# A/B kernel timing on the GPU box: ab/libsnn_lif_base.so (reference build) vs the in-tree build.
# usage: bash tools/gpu_ab.sh [cases] [pytest target]
cases=${1:-cfg1,cfg2,t16}
mkdir -p gpurun_out/ab
for i in 1 2; do
  echo "== base ($i)"; SNN_LIF_LIBRARY=$PWD/ab/libsnn_lif_base.so timeout 300 python tools/kbench.py --cases $cases
  echo "== new ($i)"; timeout 300 python tools/kbench.py --cases $cases
done
if [ -n "$2" ]; then timeout 900 python -m pytest -m gpu -x -q $2 2>&1 | tail -5; fi
