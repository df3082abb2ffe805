# ncu --set full of the cfg1 T=512 forward + backward for each library build in ab/ (A/B of DRAM traffic).
mkdir -p gpurun_out/ab
for l in "$@"; do
  SNN_LIF_LIBRARY=$PWD/ab/$l timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:lif_ --launch-skip 2 --launch-count 2 --csv python tools/prof_step.py --T 512 --N 1048576 --steps 2 > gpurun_out/ab/ncu_$l.csv 2>&1
done
