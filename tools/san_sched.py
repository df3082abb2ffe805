"""Launch-scheduling paths for compute-sanitizer (r2b): grids larger than the resident CTAs (one
steal request in flight, cluster launch control), the early L2 prefetch of short tiles before
griddepcontrol.wait (T <= 32) and long tiles without it, back to back so programmatic dependent
launch overlaps them; plus the NCCL-window handoff on a 1-rank communicator."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
from paper_2408_00280_b200 import dist as D, handoff as HO  # noqa: E402

p = snn.LIFParams.paper()
for dt in (torch.float32, torch.bfloat16):
    for T in (8, 16, 40):
        N = (1 << 20) + 1024
        x = torch.randn(T, N, device="cuda", dtype=dt)
        g = torch.randn(T, N, device="cuda", dtype=dt)
        for fmt in ("u8", "bits"):
            f = snn.lif_forward(x, p, spike_fmt=fmt)
            snn.lif_backward(g, f)
comm = D.NcclComm()
w = HO.WindowHandoff(comm, 5000)
x = torch.randn(12, 5000, device="cuda")
f = HO.lif_forward_handoff(x, p, w.forward_handoff())
HO.lif_backward_handoff(torch.randn_like(x), f, w.backward_handoff())
torch.cuda.synchronize()
w.close()
comm.close()
print("done")
