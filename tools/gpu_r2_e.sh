set -x
O=gpurun_out/r2e
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_forward --launch-skip 1 --launch-count 1 -o $O/unal_f32_fwd -f python tools/prof_step.py --T 64 --N 1048577 --steps 2 > $O/unal_f32.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_backward --launch-skip 1 --launch-count 1 -o $O/unal_bf16_bwd -f python tools/prof_step.py --T 64 --N 4194305 --dtype bf16 --steps 2 > $O/unal_bf16.log 2>&1
ls -la $O
