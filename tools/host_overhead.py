"""Host-side cost of one eager lif_forward / lif_backward call (tiny layer, GPU never the
bottleneck): wall time per call averaged over many calls, and the same for the bare C ABI
call with pre-built arguments, so the Python marshalling and the library's own host work
(validation, tensor-map encode, launch) are separated.

    python tools/host_overhead.py [--calls 2000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
from paper_2408_00280_b200 import _lib  # noqa: E402


def per_call(fn, calls):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(calls):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / calls * 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=2000)
    a = ap.parse_args()
    T, N = 16, 4096
    x = torch.randn(T, N, device="cuda")
    g = torch.randn(T, N, device="cuda")
    p = snn.LIFParams.paper()
    f = snn.lif_forward(x, p, return_v_final=False)
    out = {}
    out["lif_forward (python API)"] = per_call(lambda: snn.lif_forward(x, p, return_v_final=False), a.calls)
    out["lif_backward (python API)"] = per_call(
        lambda: snn.lif_backward(g, f, return_grad_v_init=False), a.calls)
    cp, shape = p.to_c(), f.shape
    st = torch.cuda.current_stream().cuda_stream
    sp = torch.empty(T, N, dtype=torch.uint8, device="cuda")
    gx = torch.empty_like(x)
    out["snn_lif_forward (C ABI only)"] = per_call(
        lambda: _lib.snn_lif_forward(cp, shape, x.data_ptr(), None, sp.data_ptr(), f.saved.data_ptr(),
                                     None, st), a.calls)
    out["snn_lif_backward (C ABI only)"] = per_call(
        lambda: _lib.snn_lif_backward(cp, shape, g.data_ptr(), x.data_ptr(), None, f.saved.data_ptr(),
                                      None, gx.data_ptr(), None, st), a.calls)
    xb, gb = x.clone(), g.clone()
    plan = snn.LIFPlan(xb, p, grad_spikes=gb)
    out["LIFPlan.forward (recorded launch)"] = per_call(plan.forward, a.calls)
    out["LIFPlan.backward (recorded launch)"] = per_call(plan.backward, a.calls)
    h = plan._plan
    st2 = torch.cuda.current_stream().cuda_stream
    out["snn_lif_plan_forward (C ABI only)"] = per_call(lambda: _lib.lib.snn_lif_plan_forward(h, st2), a.calls)
    layer = snn.LIFLayer(p)
    xr = torch.randn(T, N, device="cuda", requires_grad=True)

    def train_step():
        y = layer(xr)
        y.backward(g)
    out["LIFLayer forward+backward (autograd)"] = per_call(train_step, a.calls // 2)
    for k, v in out.items():
        print(f"{k:40s} {v:7.1f} us/call")


if __name__ == "__main__":
    main()
