"""Small affine-prologue runs (TMA and generic paths, ragged shapes; with and without the
residual shortcut on the TMA path) for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402

p = snn.LIFParams.paper()
for (T, B, C, HW, dt) in [(17, 2, 3, 100, torch.float32), (33, 4, 6, 100, torch.float32),
                          (16, 2, 4, 64, torch.bfloat16), (5, 3, 7, 1, torch.float32)]:
    N = B * C * HW
    x = torch.randn(T, N, device="cuda", dtype=dt)
    g = torch.randn(T, N, device="cuda", dtype=dt)
    spec = snn.AffineSpec(torch.rand(C, device="cuda") + 0.5, torch.randn(C, device="cuda"), C, HW)
    f = snn.lif_forward_affine(x, p, spec)
    snn.lif_backward_affine(g, f)
    if N % 8 == 0:   # the residual prologue runs on the TMA path only
        r = torch.randn(T, N, device="cuda", dtype=dt)
        for fmt in ("u8", "bits", "io"):
            f = snn.lif_forward_affine(x, p, spec, residual=r, spike_fmt=fmt)
            snn.lif_backward_affine(g, f)
torch.cuda.synchronize()
print("done")
