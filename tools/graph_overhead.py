"""How much of a graph-launched multi-layer step is per-kernel event recording rather than
kernel time: the cfg2 (VGG-11 bf16, T=16) step captured with and without a CUDA-event pair
around every kernel (bench.py records them for its roofline), through LIFPlans.

    python tools/graph_overhead.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
import snn_synth  # noqa: E402

VGG11 = [(64, 32, 32), (128, 16, 16), (256, 8, 8), (256, 8, 8), (512, 4, 4), (512, 4, 4), (512, 2, 2), (512, 2, 2)]


def main():
    B, T = 128, 16
    p = snn.LIFParams.paper()
    plans = []
    for i, (c, h, w) in enumerate(VGG11):
        N = B * c * h * w
        X = snn_synth.normal_tensor(1234 + i, T, N, device="cuda", dtype=torch.bfloat16)
        G = snn_synth.normal_tensor(4321 + i, T, N, device="cuda", dtype=torch.bfloat16)
        plans.append(snn.LIFPlan(X, p, grad_spikes=G))

    keep = []   # captured events must outlive the graph

    def step(events):
        for pl in plans:
            if events:
                a, b = torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)
                a.record(); pl.forward(); b.record(); keep.extend((a, b))
            else:
                pl.forward()
            if events:
                a, b = torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)
                a.record(); pl.backward(); b.record(); keep.extend((a, b))
            else:
                pl.backward()

    for events in (False, True):
        for _ in range(3):
            step(events)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                step(events)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        print(f"per-kernel events {'on ' if events else 'off'}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per step")


if __name__ == "__main__":
    main()
