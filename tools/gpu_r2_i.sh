# Round-2 evidence pass: GPU suite, bench lines (default, cfg2, cfg4, sweep, N=2 debug), ncu launch lists.
set -x
O=gpurun_out/r2i
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 400 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 400 python bench.py --sweep --serial --no-cpu-baseline --no-e2e > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 600 python bench.py --gpus 2 --debug-single-gpu --steps 3 --warmup 3 --no-e2e --tsplit-steps 3 > $O/bench_n2_debug.json 2> $O/bench_n2_debug.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg1.csv 2> $O/launches_cfg1.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --workload cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg2.csv 2> $O/launches_cfg2.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --workload cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg4.csv 2> $O/launches_cfg4.err
ls -la $O
