set -x
mkdir -p gpurun_out/p1
NCU=/usr/local/cuda/bin/ncu
timeout 300 python bench.py --workload cfg2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p1/bench_cfg2.json 2> gpurun_out/p1/bench_cfg2.err
timeout 300 python bench.py --sweep --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p1/bench_sweep.json 2> gpurun_out/p1/bench_sweep.err
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_ --launch-skip 2 --launch-count 2 -o gpurun_out/p1/bf16_T16 -f python tools/prof_step.py --T 16 --N 8388608 --dtype bf16 --steps 2 > gpurun_out/p1/ncu1.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_ --launch-skip 2 --launch-count 2 -o gpurun_out/p1/f32_T8 -f python tools/prof_step.py --T 8 --N 1048576 --dtype f32 --steps 2 > gpurun_out/p1/ncu2.log 2>&1
ls -la gpurun_out/p1
