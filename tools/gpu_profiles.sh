# Round profile refresh (1x B200): bench lines + ncu launch list + ncu full captures.
# Outputs under gpurun_out/prof/; summarised into profiles/ by tools/ncu_summary.py here.
set -x
O=gpurun_out/prof
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 400 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 300 python bench.py --sweep --serial --no-cpu-baseline --no-e2e > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg1.csv 2> $O/launches_cfg1.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --workload cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg2.csv 2> $O/launches_cfg2.err
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:lif_ -s 6 -c 2 -o $O/full_cfg1 -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/full_cfg1.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_ --launch-skip 2 --launch-count 2 -o $O/full_bf16_T16 -f python tools/prof_step.py --T 16 --N 8388608 --dtype bf16 --steps 2 > $O/full_bf16.log 2>&1
ls -la $O
