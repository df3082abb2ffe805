set -x
O=gpurun_out/r2h
mkdir -p $O
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:lif_backward --launch-skip 2 --launch-count 2 -o $O/aff_bwd -f python tools/affine_ab.py > $O/aff.log 2>&1
