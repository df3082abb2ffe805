"""Unaligned-row and ragged-N runs of the TMA kernels (1-D tensor maps, element-wise stores, a
ragged last VEC group), plain / affine / residual, every spike format, for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402

p = snn.LIFParams.paper()
for dt in (torch.float32, torch.bfloat16):
    for T in (5, 16, 37):
        for N, off in ((1027, 0), (4099, 0), (2048, 1), (1531, 3)):
            x = torch.randn(T, N + off, device="cuda", dtype=dt)[:, off:]
            g = torch.randn(T, N + off, device="cuda", dtype=dt)[:, off:]
            for save in ("recompute", "h"):
                for fmt in ("u8", "bits", "io"):
                    f = snn.lif_forward(x, p, save_mode=save, spike_fmt=fmt,
                                        v_init=torch.randn(N, device="cuda"))
                    snn.lif_backward(g, f, grad_v_final=torch.randn(N, device="cuda"))
            if off == 0:
                C = 1
                HW = N
                spec = snn.AffineSpec(torch.rand(C, device="cuda") + 0.5, torch.randn(C, device="cuda"), C, HW)
                r = torch.randn(T, N, device="cuda", dtype=dt)
                f = snn.lif_forward_affine(x, p, spec, residual=r)
                snn.lif_backward_affine(g, f)
torch.cuda.synchronize()
print("done")
