# r2c: executed SASS opcodes of the aligned vs unaligned fp32 forward (T=64, N=2^22 / 2^22+1).
O=gpurun_out/r2c_ops; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
for c in "al_f32 --N 4194304" "unal_f32 --N 4194305"; do
  set -- $c; n=$1; shift
  timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_forward --launch-skip 1 --launch-count 1 -o /tmp/$n -f python tools/prof_step.py --T 64 --steps 2 "$@" > $O/$n.log 2>&1
  python tools/ncu_opcodes.py /tmp/$n.ncu-rep lif_forward 40 > $O/${n}_ops.txt 2>&1
  $NCU -i /tmp/$n.ncu-rep --page source --csv --print-source sass --kernel-name regex:lif_forward > $O/${n}_sass.csv 2>/dev/null
  gzip -f $O/${n}_sass.csv
  rm -f /tmp/$n.ncu-rep
done
ls -la $O
