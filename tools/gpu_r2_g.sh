set -x
O=gpurun_out/r2g
mkdir -p $O
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/affine_ab.py > $O/affine_launches.csv 2> $O/affine.err
