# r2c-b: new checkpoint tests, fp32 forward tile-geometry A/B (clean flush), sweep with the clean flush.
O=gpurun_out/r2c_b; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_ckpt.py tests/test_gpu_comm.py tests/test_gpu_handoff.py -q -p no:cacheprovider -rs > $O/pytest_ckpt.log 2>&1; echo "rc=$?" >> $O/pytest_ckpt.log
for v in default w512 w256; do
  if [ $v = default ]; then L=""; else L=paper_2408_00280_b200/build_$v/libsnn_lif_$v.so; fi
  echo "== $v" >> $O/tiles.log
  SNN_LIF_LIBRARY=$L timeout 300 python tools/small_t_probe.py --T 8,16,32,128,512 --preps clean --families tma >> $O/tiles.log 2>&1
done
timeout 400 python bench.py --sweep --serial --no-cpu-baseline --no-e2e > $O/bench_sweep.json 2> $O/bench_sweep.err
