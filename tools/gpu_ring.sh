# Ring-depth sweep (SNN_LIF_RING_FWD / _BWD) on short-T shapes.
mkdir -p gpurun_out/ab
for r in 0 1 2 3 4; do
  echo "== ring fwd=$r bwd=$r (0 = configured)"
  SNN_LIF_RING_FWD=$r SNN_LIF_RING_BWD=$r timeout 300 python tools/kbench.py --cases short,cfg1
done
timeout 600 python -m pytest -m gpu -x -q tests/test_gpu_parity.py tests/test_gpu_handoff.py 2>&1 | tail -3
SNN_LIF_RING_FWD=1 SNN_LIF_RING_BWD=1 timeout 600 python -m pytest -m gpu -x -q tests/test_gpu_parity.py tests/test_gpu_handoff.py 2>&1 | tail -3
