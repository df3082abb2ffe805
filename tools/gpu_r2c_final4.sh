# Round-2c closing pass (after the unaligned forward + backward changes): GPU suite, smoke, default + cfg2 + sweep lines, one
# ncu --set full of the dominant kernel (summarised on the box: the merge-back limit is 64 MiB).
set -x
O=gpurun_out/r2cx; mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 400 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_backward --launch-skip 1 --launch-count 1 -o /tmp/full_cfg1_bwd -f python tools/prof_step.py --T 512 --N 1048576 --steps 2 > $O/full_cfg1_bwd.log 2>&1
python tools/ncu_summary.py full /tmp/full_cfg1_bwd.ncu-rep $O/full_cfg1_bwd.md --kernel lif_backward --traffic-key cfg1_T512_recompute_u8_bwd > /dev/null 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
python tools/ncu_stalls.py /tmp/full_cfg1_bwd.ncu-rep > $O/full_cfg1_bwd_stalls.txt 2>&1
rm -f /tmp/full_cfg1_bwd.ncu-rep
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg1.csv 2> $O/launches_cfg1.err
ls -la $O
timeout 600 python tools/kbench.py --cases unal --reps 20 > $O/kbench_unal.log 2>&1
timeout 400 python bench.py --sweep --serial --no-cpu-baseline --no-e2e > $O/bench_sweep.json 2> $O/bench_sweep.err
