mkdir -p gpurun_out/p2
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_ --launch-skip 4 --launch-count 2 -o gpurun_out/p2/bf16_T16_small -f python tools/prof_step.py --T 16 --N 262144 --dtype bf16 --steps 3 > gpurun_out/p2/ncu1.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg --clock-control none python tools/prof_step.py --T 1 --N 16384 --dtype bf16 --steps 3 > gpurun_out/p2/ncu_tiny.log 2>&1
