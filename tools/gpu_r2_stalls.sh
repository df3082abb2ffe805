# ncu --set full of the small-T / small-layer kernels (cfg1 T=8, T=32; cfg2 conv5 1M and conv7 262K
# neurons, bf16 T=16): stall breakdowns + metric summaries (text only; the reports stay on the box).
set -x
O=gpurun_out/r2st
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
run() {  # name, prof_step args...
  n=$1; shift
  timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_ --launch-skip 2 --launch-count 2 -o $O/$n -f python tools/prof_step.py --steps 2 "$@" > $O/$n.log 2>&1
  python tools/ncu_stalls.py $O/$n.ncu-rep > $O/$n.stalls.txt 2>&1
  python tools/ncu_summary.py full $O/$n.ncu-rep $O/$n.md > /dev/null 2>&1
  rm -f $O/$n.ncu-rep
}
run f32_T8 --T 8 --N 1048576
run f32_T32 --T 32 --N 1048576
run bf16_T16_1M --T 16 --N 1048576 --dtype bf16
run bf16_T16_262K --T 16 --N 262144 --dtype bf16
ls -la $O
