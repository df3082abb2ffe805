# r2c: u8 spikes of unaligned bf16 rows as two predicated u8x4 stores -- tests + kbench.
O=gpurun_out/r2c_unal4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_handoff.py tests/test_gpu_ckpt.py tests/test_gpu_sched.py -q -p no:cacheprovider -rs -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/kbench.py --cases unal --reps 20 > $O/kbench_unal.log 2>&1
