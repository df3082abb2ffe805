"""Ragged-T / ragged-N runs of the TMA kernels (masked and half-chunk backward paths, guarded
forward stages), plain / affine / residual, for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402

p = snn.LIFParams.paper()
for dt in (torch.float32, torch.bfloat16):
    for T in (4, 8, 10, 20, 37):
        for N in (1024 + 512 + 8, 4096):        # a ragged last tile and full tiles
            x = torch.randn(T, N, device="cuda", dtype=dt)
            g = torch.randn(T, N, device="cuda", dtype=dt)
            for save in ("recompute", "h"):
                f = snn.lif_forward(x, p, save_mode=save)
                snn.lif_backward(g, f, grad_v_final=torch.randn(N, device="cuda"))
            C, HW = 8, N // 8
            spec = snn.AffineSpec(torch.rand(C, device="cuda") + 0.5, torch.randn(C, device="cuda"), C, HW)
            r = torch.randn(T, N, device="cuda", dtype=dt)
            f = snn.lif_forward_affine(x, p, spec, residual=r)
            snn.lif_backward_affine(g, f)
torch.cuda.synchronize()
print("done")
