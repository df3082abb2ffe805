# Unaligned-row TMA kernels with warp-wide TMA issue: tests + kbench + memcheck.
set -x
O=gpurun_out/r2d
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_handoff.py tests/test_gpu_comm.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python tools/kbench.py --cases unal > $O/kbench.log 2>&1
timeout 900 $CS --tool memcheck --print-limit 20 python tools/san_unaligned.py > $O/san.log 2>&1; echo "rc=$?" >> $O/san.log
timeout 900 $CS --tool synccheck --print-limit 20 python tools/san_unaligned.py >> $O/san.log 2>&1; echo "rc=$?" >> $O/san.log
