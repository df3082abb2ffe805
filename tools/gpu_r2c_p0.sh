# r2c: bf16 plain forward with the paper-mode (P0) charge -- A/B vs SNN_BF16_FWD_P0=0, tests.
O=gpurun_out/r2c_p0; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_ckpt.py -q -p no:cacheprovider -rs -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
for v in default nop0; do
  if [ $v = default ]; then L=""; else L=paper_2408_00280_b200/build_$v/libsnn_lif_$v.so; fi
  echo "== $v" >> $O/kbench.log
  SNN_LIF_LIBRARY=$L timeout 300 python tools/kbench.py --cases cfg2 --reps 20 >> $O/kbench.log 2>&1
  SNN_LIF_LIBRARY=$L timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2_${v}_$i.json 2> $O/bench_cfg2_${v}_$i.err
done
done
