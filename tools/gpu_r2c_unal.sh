# r2c: realigned 16-byte shared-memory loads on the unaligned-row kernels -- tests + kbench.
O=gpurun_out/r2c_unal; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_handoff.py tests/test_gpu_ckpt.py -q -p no:cacheprovider -rs > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/kbench.py --cases unal --reps 20 > $O/kbench_unal.log 2>&1
timeout 600 python tools/kbench.py --cases unal --reps 20 > $O/kbench_unal2.log 2>&1
