"""Time lif_fwd_bwd_host (host-buffer path) at cfg1 T=512 for several chunk sizes / slot counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402

T, N = 512, 1 << 20
p = snn.LIFParams.paper()
X = torch.randn(T, N).pin_memory()
G = torch.randn(T, N).pin_memory()
S = torch.empty(T, N, dtype=torch.uint8).pin_memory()
GX = torch.empty(T, N).pin_memory()
# naive: one copy each way on one stream
xd = X.cuda(); torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    xd = X.to("cuda", non_blocking=True); gd = G.to("cuda", non_blocking=True)
    f = snn.lif_forward(xd, p); gx, _ = snn.lif_backward(gd, f)
    S.copy_(f.spikes, non_blocking=True); GX.copy_(gx, non_blocking=True)
    torch.cuda.synchronize()
    print("naive", round((time.perf_counter() - t0) * 1e3, 1), "ms", flush=True)
del xd, gd, f, gx
for chunk in (8192, 16384, 32768, 65536):
    for ns in (2, 3, 4):
        ws = snn.host_workspace(T, N, p, chunk_neurons=chunk, nslots=ns)
        snn.lif_fwd_bwd_host(X, G, p, spikes=S, grad_x=GX, chunk_neurons=chunk, nslots=ns, workspace=ws)
        ts = []
        for rep in range(3):
            t0 = time.perf_counter()
            snn.lif_fwd_bwd_host(X, G, p, spikes=S, grad_x=GX, chunk_neurons=chunk, nslots=ns, workspace=ws)
            ts.append(time.perf_counter() - t0)
        print("chunk", chunk, "slots", ns, "ms", round(min(ts) * 1e3, 1), flush=True)
        del ws
