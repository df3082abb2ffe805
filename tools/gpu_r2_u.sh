# Unaligned rows: 16-B smem row pitch, widest smem loads, funnel-shift u8 spike stores.
set -x
O=gpurun_out/r2u
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python tools/kbench.py --cases unal > $O/kbench_unal.log 2>&1
ls -la $O
