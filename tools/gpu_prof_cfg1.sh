# cfg1 (default bench workload) launch list + ncu full capture, for profiles/.
O=gpurun_out/prof; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg1.csv 2> $O/launches_cfg1.err
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:lif_ -s 6 -c 2 -o $O/full_cfg1 -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/full_cfg1.log 2>&1
timeout 300 python bench.py --sweep --serial --no-cpu-baseline --no-e2e > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
ls -la $O
