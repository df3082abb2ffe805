# Unaligned rows through LDGSTS (whole producer warp) instead of per-row bulk copies.
set -x
O=gpurun_out/r2aa
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "unal or ragged or golden or handoff or residual" > $O/pytest_unal.log 2>&1; echo "rc=$?" >> $O/pytest_unal.log
timeout 300 python tools/kbench.py --cases unal > $O/kbench_unal.log 2>&1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 10 python tools/san_unaligned.py > $O/san_memcheck.log 2>&1; echo "rc=$?" >> $O/san_memcheck.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool synccheck --print-limit 10 python tools/san_unaligned.py > $O/san_synccheck.log 2>&1; echo "rc=$?" >> $O/san_synccheck.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 10 python tools/san_unaligned.py > $O/san_racecheck.log 2>&1; echo "rc=$?" >> $O/san_racecheck.log
ls -la $O
