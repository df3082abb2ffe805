"""Plain LIF vs the fused affine prologue on one layer (bench.py --affine's shape), a few
steps each -- for an ncu launch list (per-kernel durations) of the prologue's cost.

    ncu --metrics gpu__time_duration.sum --clock-control none python tools/affine_ab.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
import snn_synth  # noqa: E402

T, B, C, HW = 64, 16, 64, 1024
N = B * C * HW
p = snn.LIFParams.paper()
X = snn_synth.normal_tensor(1234, T, N, device="cuda")
G = snn_synth.normal_tensor(4321, T, N, device="cuda")
spec = snn.AffineSpec(torch.linspace(0.5, 1.5, C, device="cuda"), torch.linspace(-0.2, 0.2, C, device="cuda"), C, HW)
for _ in range(3):
    f = snn.lif_forward(X, p, return_v_final=False)
    snn.lif_backward(G, f, return_grad_v_init=False)
    f = snn.lif_forward_affine(X, p, spec, return_v_final=False)
    snn.lif_backward_affine(G, f, return_grad_v_init=False)
torch.cuda.synchronize()
print("done")
