"""RECOMPUTE without the V[-1] checkpoint (r2c) for compute-sanitizer: v_init given / absent,
T <= 16 (no checkpoint at all) and T > 16, ragged last tile, both kernel families, the affine
pair with v_init, and a 1-rank NCCL time split (the backward re-reads v_in_ws)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
from paper_2408_00280_b200 import dist as D  # noqa: E402

p = snn.LIFParams.paper()
for fam in ("0", "1"):
    os.environ["SNN_LIF_NO_TMA"] = fam
    for dt in (torch.float32, torch.bfloat16):
        for T in (1, 8, 16, 17, 40):
            N = 5000 + 8
            x = torch.randn(T, N, device="cuda", dtype=dt)
            g = torch.randn(T, N, device="cuda", dtype=dt)
            for v0 in (None, torch.randn(N, device="cuda")):
                f = snn.lif_forward(x, p, v_init=v0)
                snn.lif_backward(g, f)
    C, HW, B = 8, 64, 4
    af = snn.AffineSpec(torch.rand(C, device="cuda") + 0.5, torch.randn(C, device="cuda"), C, HW)
    x = torch.randn(12, B * C * HW, device="cuda")
    f = snn.lif_forward_affine(x, p, af, v_init=torch.randn(B * C * HW, device="cuda"))
    snn.lif_backward_affine(torch.randn_like(x), f)
os.environ["SNN_LIF_NO_TMA"] = "0"
comm = D.NcclComm()
x = torch.randn(20, 6000, device="cuda")
f = D.lif_forward_tsplit(comm, x, p, n_chunks=4, v_init=torch.randn(6000, device="cuda"))
D.lif_backward_tsplit(comm, torch.randn_like(x), f, n_chunks=4)
torch.cuda.synchronize()
comm.close()
print("done")
