set -x
O=gpurun_out/r2k
mkdir -p $O
timeout 300 python tools/launch_overhead.py > $O/lo_pdl.log 2>&1
SNN_LIF_NO_PDL=1 timeout 300 python tools/launch_overhead.py > $O/lo_nopdl.log 2>&1
timeout 400 python bench.py --sweep --no-cpu-baseline --no-e2e --steps 5 > $O/bench_sweep.json 2> $O/bench_sweep.err
timeout 400 python bench.py --workload cfg3 --steps 5 --no-e2e > $O/bench_cfg3_k1.json 2> $O/bench_cfg3_k1.err
