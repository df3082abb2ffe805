# Sweep bench line + bf16 T=512 backward and cfg1 T=8 ncu captures, for profiles/ (1x B200).
O=gpurun_out/prof; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 300 python bench.py --sweep --serial --no-cpu-baseline --no-e2e > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_backward --launch-skip 1 --launch-count 1 -o $O/full_bf16_T512 -f python tools/prof_step.py --T 512 --N 1048576 --dtype bf16 --steps 2 > $O/full_bf16_T512.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_ --launch-skip 2 --launch-count 2 -o $O/full_f32_T8 -f python tools/prof_step.py --T 8 --N 1048576 --dtype f32 --steps 2 > $O/full_f32_T8.log 2>&1
ls -la $O
