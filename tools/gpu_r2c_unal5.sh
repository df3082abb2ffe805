# r2c: branch-free unaligned loads / predicated stores in the backward (fp32 and bf16 pairs) -- tests + kbench.
O=gpurun_out/r2c_unal5; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_handoff.py tests/test_gpu_ckpt.py tests/test_gpu_sched.py -q -p no:cacheprovider -rs -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/kbench.py --cases unal --reps 20 > $O/kbench_unal.log 2>&1
timeout 600 python tools/kbench.py --cases unal --reps 20 > $O/kbench_unal2.log 2>&1
