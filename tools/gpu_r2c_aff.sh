# r2c: plain vs affine forward/backward (T=64, N=1M, C=64): ncu durations, opcode mix.
O=gpurun_out/r2c_aff; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
for c in "plain" "aff --affine-c 64"; do
  set -- $c; n=$1; shift
  timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_ --launch-skip 2 --launch-count 2 -o /tmp/$n -f python tools/prof_step.py --T 64 --N 1048576 --steps 3 "$@" > $O/$n.log 2>&1
  python tools/ncu_opcodes.py /tmp/$n.ncu-rep lif_forward 25 > $O/${n}_fwd_ops.txt 2>&1
  python tools/ncu_opcodes.py /tmp/$n.ncu-rep lif_backward 25 > $O/${n}_bwd_ops.txt 2>&1
  python tools/ncu_stalls.py /tmp/$n.ncu-rep > $O/${n}_stalls.txt 2>&1
  python tools/ncu_summary.py full /tmp/$n.ncu-rep $O/${n}_full.md --kernel lif_ > /dev/null 2>&1
  rm -f /tmp/$n.ncu-rep
done
