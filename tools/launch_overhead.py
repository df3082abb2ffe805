"""Per-launch cost of the fused kernels on small layers, back to back inside a CUDA graph
(the same launch repeated, so the inputs stay L2-resident: what remains is the per-launch
fixed cost plus L2 traffic).  Set SNN_LIF_NO_PDL=1 to launch without programmatic dependent
launch for an A/B.

    python tools/launch_overhead.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
import snn_synth  # noqa: E402

p = snn.LIFParams.paper()
REPS = 50


def per_launch(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(REPS):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / REPS * 1e3


z = torch.zeros(1, device="cuda")
print(f"torch add_ on 1 element: {per_launch(lambda: z.add_(1.0)):.2f} us per launch", flush=True)
for dt, T, N in [(torch.bfloat16, 16, 1 << 18), (torch.bfloat16, 16, 1 << 20), (torch.bfloat16, 16, 1 << 21),
                 (torch.float32, 8, 1 << 20), (torch.float32, 16, 1 << 14)]:
    x = snn_synth.normal_tensor(1, T, N, device="cuda", dtype=dt)
    gs = snn_synth.normal_tensor(2, T, N, device="cuda", dtype=dt)
    f = snn.lif_forward(x, p, return_v_final=False)
    gx, _ = snn.lif_backward(gs, f, return_grad_v_init=False)
    tf = per_launch(lambda: snn.lif_forward(x, p, spikes=f.spikes, saved=f.saved, return_v_final=False))
    tb = per_launch(lambda: snn.lif_backward(gs, f, grad_x=gx, return_grad_v_init=False))
    print(f"{str(dt)[6:]:9s} T={T:3d} N={N:8d}  fwd {tf:6.2f} us  bwd {tb:6.2f} us  (L2-resident inputs)", flush=True)
