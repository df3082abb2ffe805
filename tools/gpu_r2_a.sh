# Round-2 first GPU pass: full GPU suite, the 4*sens A/B, baseline kernel timings, small-T ncu captures.
set -x
O=gpurun_out/r2a
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
PARITY_SENS=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_handoff.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > $O/pytest_sens0.log 2>&1; echo "rc=$?" >> $O/pytest_sens0.log
timeout 300 python tools/kbench.py --cases sweep,cfg2,small > $O/kbench.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_ --launch-skip 2 --launch-count 2 -o $O/full_T8 -f python tools/prof_step.py --T 8 --N 1048576 --steps 2 > $O/full_T8.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_ --launch-skip 2 --launch-count 2 -o $O/full_T32 -f python tools/prof_step.py --T 32 --N 1048576 --steps 2 > $O/full_T32.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:lif_ --launch-skip 2 --launch-count 2 -o $O/full_bf16_262k -f python tools/prof_step.py --T 16 --N 262144 --dtype bf16 --steps 2 > $O/full_262k.log 2>&1
ls -la $O
