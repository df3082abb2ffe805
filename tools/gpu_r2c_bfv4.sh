# r2c: bf16 forward geometry VEC 4 x 256 lanes vs the default VEC 8 x 128 at cfg2 (two rounds).
O=gpurun_out/r2c_bfv4; mkdir -p $O
for i in 1 2; do
for v in default bfv4; do
  if [ $v = default ]; then L=""; else L=paper_2408_00280_b200/build_$v/libsnn_lif_$v.so; fi
  SNN_LIF_LIBRARY=$L timeout 300 python bench.py --workload cfg2 --no-cpu-baseline --no-e2e > $O/bench_cfg2_${v}_$i.json 2> $O/bench_cfg2_${v}_$i.err
done
done
