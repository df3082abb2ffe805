# ncu full captures: fp32 forward aligned vs unaligned rows (T=64), bf16 backward unaligned.
set -x
O=gpurun_out/r2t
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_forward --launch-skip 1 --launch-count 1 -o $O/al_f32_fwd -f python tools/prof_step.py --T 64 --N 1048576 --steps 2 > $O/al_f32.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_forward --launch-skip 1 --launch-count 1 -o $O/unal_f32_fwd -f python tools/prof_step.py --T 64 --N 1048577 --steps 2 > $O/unal_f32.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_backward --launch-skip 1 --launch-count 1 -o $O/unal_f32_bwd -f python tools/prof_step.py --T 64 --N 1048577 --steps 2 > $O/unal_f32b.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_backward --launch-skip 1 --launch-count 1 -o $O/unal_bf16_bwd -f python tools/prof_step.py --T 64 --N 4194305 --dtype bf16 --steps 2 > $O/unal_bf16.log 2>&1
ls -la $O
for r in al_f32_fwd unal_f32_fwd unal_f32_bwd unal_bf16_bwd; do
  python tools/ncu_stalls.py $O/$r.ncu-rep > $O/$r.stalls.txt 2>&1
  python tools/ncu_hot.py $O/$r.ncu-rep lif_ 45 > $O/$r.hot.txt 2>&1
  $NCU -i $O/$r.ncu-rep --page details --csv > $O/$r.details.csv 2>&1
  rm -f $O/$r.ncu-rep
done
ls -la $O
