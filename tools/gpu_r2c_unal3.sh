# r2c: branch-free unaligned 16-byte smem loads + predicated u8x4 spike stores -- tests + kbench.
O=gpurun_out/r2c_unal3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_handoff.py tests/test_gpu_ckpt.py tests/test_gpu_sched.py -q -p no:cacheprovider -rs -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/kbench.py --cases unal --reps 20 > $O/kbench_unal.log 2>&1
timeout 600 python tools/kbench.py --cases unal --reps 20 --spike-fmt bits > $O/kbench_unal_bits.log 2>&1
