# Round-2c evidence pass on the final tree: GPU suite, smoke, bench lines, ncu launch lists with
# DRAM bytes, one ncu --set full of the dominant kernel, sanitizers on the checkpoint change.
set -x
O=gpurun_out/r2cf
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
CS=/usr/local/cuda/bin/compute-sanitizer
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 400 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --no-e2e > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 300 python bench.py --workload cfg4 --prologue --no-cpu-baseline --no-e2e > $O/bench_cfg4_prologue.json 2> $O/bench_cfg4_prologue.err
timeout 600 python bench.py --steps 5 --warmup 3 --T 32 --no-e2e --no-cpu-baseline --affine --prologue > $O/bench_affine.json 2> $O/bench_affine.err
timeout 400 python bench.py --sweep --serial --no-cpu-baseline --no-e2e > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 400 python bench.py --workload cfg3 --steps 5 --no-e2e > $O/bench_cfg3_k1.json 2> $O/bench_cfg3_k1.err
timeout 600 python bench.py --gpus 2 --debug-single-gpu --steps 3 --warmup 3 --no-e2e --tsplit-steps 3 > $O/bench_n2_debug.json 2> $O/bench_n2_debug.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg1.csv 2> $O/launches_cfg1.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --workload cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg2.csv 2> $O/launches_cfg2.err
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:lif_ --csv python bench.py --workload cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > $O/launches_cfg4.csv 2> $O/launches_cfg4.err
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_backward --launch-skip 2 --launch-count 1 -o $O/full_cfg1_bwd -f python tools/prof_step.py --T 512 --N 1048576 --steps 2 > $O/full_cfg1_bwd.log 2>&1
for tool in memcheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 10 python tools/san_ckpt.py > $O/san_ckpt_$tool.log 2>&1
  echo "rc=$?" >> $O/san_ckpt_$tool.log
done
ls -la $O
