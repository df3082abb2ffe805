# bf16 forward tile geometry A/B: VEC 8 x 128 lanes (base) vs VEC 4 x 256 lanes (v4).
set -x
O=gpurun_out/r2ai
mkdir -p $O
for v in base v4 base2 v42; do
  case $v in base*) unset SNN_LIF_LIBRARY;; *) export SNN_LIF_LIBRARY=paper_2408_00280_b200/build_v4/libsnn_lif_v4.so;; esac
  timeout 300 python bench.py --workload cfg2 --no-e2e --no-cpu-baseline > $O/cfg2_$v.json 2> $O/cfg2_$v.err
done
unset SNN_LIF_LIBRARY; timeout 300 python tools/kbench.py --cases cfg2,bf512 > $O/kbench_base.log 2>&1
SNN_LIF_LIBRARY=paper_2408_00280_b200/build_v4/libsnn_lif_v4.so timeout 300 python tools/kbench.py --cases cfg2,bf512 > $O/kbench_v4.log 2>&1
ls -la $O
