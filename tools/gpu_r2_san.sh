# compute-sanitizer over every kernel family of round 2 (aligned / unaligned TMA, affine fold, residual, time split).
O=gpurun_out/r2san
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for w in san_ragged san_unaligned san_affine san_tsplit; do
  for tool in memcheck synccheck initcheck racecheck; do
    echo "== $w $tool" >> $O/san.log
    timeout 900 $CS --tool $tool --print-limit 10 python tools/$w.py > $O/${w}_${tool}.log 2>&1
    echo "rc=$?" >> $O/san.log
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Hazard|done" $O/${w}_${tool}.log | tail -4 >> $O/san.log
  done
done
