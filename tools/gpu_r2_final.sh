# Round-2b evidence pass on the final tree: GPU suite, bench lines, launch lists with DRAM bytes,
# per-CTA timelines, sanitizers on the new scheduling / window paths.
set -x
O=gpurun_out/r2f
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
CS=/usr/local/cuda/bin/compute-sanitizer
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 400 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 300 python bench.py --workload cfg4 --prologue --no-cpu-baseline --no-e2e > $O/bench_cfg4_prologue.json 2> $O/bench_cfg4_prologue.err
timeout 400 python bench.py --sweep --serial --no-cpu-baseline --no-e2e > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 600 python bench.py --gpus 2 --debug-single-gpu --steps 3 --warmup 3 --no-e2e --tsplit-steps 3 > $O/bench_n2_debug.json 2> $O/bench_n2_debug.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg1.csv 2> $O/launches_cfg1.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --workload cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg2.csv 2> $O/launches_cfg2.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --workload cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg4.csv 2> $O/launches_cfg4.err
timeout 300 python tools/trace_timeline.py --scenario cfg2,t8,t8flush,t32,t512 --reps 1 --order > $O/timeline.log 2>&1
for tool in memcheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 10 python tools/san_sched.py > $O/san_sched_$tool.log 2>&1
  echo "rc=$?" >> $O/san_sched_$tool.log
done
ls -la $O
