"""Run a few fused LIF fwd+bwd steps for ncu / sanitizer captures (no timing, no oracle).

    python tools/prof_step.py [--T 512] [--N 1048576] [--dtype f32|bf16] [--save-mode recompute|h]
                              [--spike-fmt u8|bits|io] [--steps 3] [--affine-c C]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
import snn_synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=512)
    ap.add_argument("--N", type=int, default=1 << 20)
    ap.add_argument("--dtype", choices=["f32", "bf16"], default="f32")
    ap.add_argument("--save-mode", default="recompute")
    ap.add_argument("--spike-fmt", default="u8")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--affine-c", type=int, default=0,
                    help="> 0: run the fused affine prologue with C channels (HW = N / (16 C))")
    a = ap.parse_args()
    dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    X = snn_synth.normal_tensor(1234, a.T, a.N, device="cuda", dtype=dt)
    G = snn_synth.normal_tensor(4321, a.T, a.N, device="cuda", dtype=dt)
    p = snn.LIFParams.paper()
    spec = None
    if a.affine_c:
        C = a.affine_c
        spec = snn.AffineSpec(torch.rand(C, device="cuda") + 0.5, torch.randn(C, device="cuda"), C,
                              a.N // (16 * C))
    for _ in range(a.steps):
        if spec is not None:
            f = snn.lif_forward_affine(X, p, spec, spike_fmt=a.spike_fmt, return_v_final=False)
            snn.lif_backward_affine(G, f, return_grad_v_init=False)
            continue
        f = snn.lif_forward(X, p, spike_fmt=a.spike_fmt, save_mode=a.save_mode, return_v_final=False)
        snn.lif_backward(G, f, return_grad_v_init=False)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
