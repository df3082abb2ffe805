mkdir -p gpurun_out/ab
echo "== TMA"; timeout 300 python tools/kbench.py --cases small,cfg2
echo "== generic (SNN_LIF_NO_TMA=1)"; SNN_LIF_NO_TMA=1 timeout 300 python tools/kbench.py --cases small,cfg2
