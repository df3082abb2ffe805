# r2c: bf16 vs fp32 aligned forward at cfg2's largest layer shape (T=16, N=8M): stalls + opcode mix.
O=gpurun_out/r2c_bf16; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
for c in "bf16_fwd --dtype bf16" "f32_fwd --dtype f32"; do
  set -- $c; n=$1; shift
  timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_forward --launch-skip 1 --launch-count 1 -o /tmp/$n -f python tools/prof_step.py --T 16 --N 8388608 --steps 2 "$@" > $O/$n.log 2>&1
  python tools/ncu_opcodes.py /tmp/$n.ncu-rep lif_forward 40 > $O/${n}_ops.txt 2>&1
  python tools/ncu_stalls.py /tmp/$n.ncu-rep > $O/${n}_stalls.txt 2>&1
  python tools/ncu_summary.py full /tmp/$n.ncu-rep $O/${n}_full.md --kernel lif_forward > /dev/null 2>&1
  python tools/ncu_hot.py /tmp/$n.ncu-rep lif_forward 30 > $O/${n}_hot.txt 2>&1
  rm -f /tmp/$n.ncu-rep
done
timeout 300 python tools/kbench.py --cases cfg2 --reps 20 > $O/kbench_cfg2.log 2>&1
