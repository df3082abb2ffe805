"""The C-ABI time split on a 1-rank NCCL communicator (chunked kernels over column windows of
the layer, u8 / bits / io spikes, both save modes) for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
from paper_2408_00280_b200 import dist as D  # noqa: E402

p = snn.LIFParams.paper()
comm = D.NcclComm()
for T, N, M in ((17, 5001, 4), (33, 12288, 7)):
    x = torch.randn(T, N, device="cuda")
    g = torch.randn(T, N, device="cuda")
    for fmt, save in (("u8", "recompute"), ("bits", "h"), ("io", "recompute")):
        f = D.lif_forward_tsplit(comm, x, p, n_chunks=M, spike_fmt=fmt, save_mode=save,
                                 v_init=torch.randn(N, device="cuda"))
        D.lif_backward_tsplit(comm, g, f, n_chunks=M, grad_v_final=torch.randn(N, device="cuda"))
torch.cuda.synchronize()
comm.close()
print("done")
