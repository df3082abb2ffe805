# r2c: unaligned forward -- kbench, ncu --set full (source) of the aligned and unaligned fp32 forward
# and the unaligned bf16 forward; reports summarised on the box (tools/ncu_hot.py, ncu_stalls.py)
# and deleted (the merge-back limit is 64 MiB).
O=gpurun_out/r2c_unal2; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 600 python tools/kbench.py --cases unal --reps 20 > $O/kbench_unal.log 2>&1
for c in "al_f32 --N 4194304" "unal_f32 --N 4194305" "unal_bf16 --N 4194305 --dtype bf16"; do
  set -- $c; n=$1; shift
  timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_forward --launch-skip 1 --launch-count 1 -o /tmp/$n -f python tools/prof_step.py --T 64 --steps 2 "$@" > $O/$n.log 2>&1
  python tools/ncu_hot.py /tmp/$n.ncu-rep lif_forward 45 > $O/${n}_hot.txt 2>&1
  python tools/ncu_stalls.py /tmp/$n.ncu-rep > $O/${n}_stalls.txt 2>&1
  python tools/ncu_summary.py full /tmp/$n.ncu-rep $O/${n}_full.md --kernel lif_forward > /dev/null 2>&1
  rm -f /tmp/$n.ncu-rep
done
ls -la $O
