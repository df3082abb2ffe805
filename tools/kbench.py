"""Per-kernel timing of the fused LIF forward / backward on a list of shapes (tuning aid, not
the bench contract): CUDA events around each launch on the launch stream, two input batches
alternated so consecutive launches do not hit each other's data in L2, algorithmic bytes
per DESIGN.md section 6.

    python tools/kbench.py [--reps 20] [--cases cfg1,cfg2,t16]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
import snn_synth  # noqa: E402

CASES = {
    "cfg1": [("f32", 512, 1 << 20)],
    "sweep": [("f32", 8, 1 << 20), ("f32", 32, 1 << 20), ("f32", 128, 1 << 20)],
    "cfg2": [("bf16", 16, 128 * 64 * 32 * 32), ("bf16", 16, 128 * 128 * 16 * 16),
             ("bf16", 16, 128 * 256 * 8 * 8), ("bf16", 16, 128 * 512 * 4 * 4),
             ("bf16", 16, 128 * 512 * 2 * 2)],
    "t16": [("f32", 16, 1 << 23)],
    "bf512": [("bf16", 512, 1 << 20)],
    "short": [("f32", 8, 1 << 20), ("f32", 16, 1 << 20), ("f32", 16, 1 << 23), ("bf16", 16, 1 << 23),
              ("bf16", 16, 1 << 21), ("f32", 64, 1 << 22)],
    "ragged": [("f32", 4, 1 << 21), ("f32", 10, 1 << 21), ("f32", 16, 1 << 21), ("f32", 20, 1 << 21),
               ("f32", 32, 1 << 21), ("bf16", 10, 1 << 22), ("bf16", 16, 1 << 22)],
    # unaligned rows (1-D tensor-map TMA kernels) vs the aligned shape: (dtype, T, N[, view offset])
    "unal": [("f32", 512, 1 << 20), ("f32", 512, (1 << 20) + 1), ("f32", 512, (1 << 20) + 2),
             ("f32", 512, (1 << 20) + 3), ("f32", 512, 1 << 20, 1), ("bf16", 64, 1 << 22),
             ("bf16", 64, (1 << 22) + 1), ("bf16", 64, 1 << 22, 3)],
    "small": [("bf16", 16, 1 << 14), ("bf16", 16, 1 << 16), ("bf16", 16, 1 << 18), ("bf16", 1, 1 << 14),
              ("f32", 16, 1 << 18), ("f32", 1, 1 << 14)],
}


def time_null(reps):
    """Event-to-event time of a trivial kernel under the same queueing (the floor)."""
    b = torch.zeros(1, device="cuda")
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda._sleep(int(2e6))
    for e0, e1 in ev:
        e0.record(st)
        b.add_(1.0)
        e1.record(st)
    torch.cuda.synchronize()
    t = sorted(e0.elapsed_time(e1) for e0, e1 in ev)[reps // 2]
    print(f"null kernel (torch add_ on 1 element): {t * 1e3:.1f} us", flush=True)


def alg_bytes(dt, T, N, save_mode="recompute"):
    e = 4 if dt == "f32" else 2
    ck = 4.0 * (-(-T // 16) - 1) / T   # checkpoint rows after the first (V[-1] is not stored)
    return (e + 1 + ck) * T * N, (3 * e + ck) * T * N


SAVE_MODE = "recompute"
SPIKE_FMT = "u8"


def time_case(dt, T, N, reps, off=0):
    """off > 0: x / grad_spikes are column views [:, off:] of [T, N + off] tensors (unaligned rows)."""
    dtype = torch.float32 if dt == "f32" else torch.bfloat16
    p = snn.LIFParams.paper()
    xs = [snn_synth.normal_tensor(1234 + i, T, N + off, device="cuda", dtype=dtype)[:, off:] for i in range(2)]
    gs = [snn_synth.normal_tensor(4321 + i, T, N + off, device="cuda", dtype=dtype)[:, off:] for i in range(2)]
    st = torch.cuda.current_stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(reps)]
    for i in range(3):
        f = snn.lif_forward(xs[i % 2], p, return_v_final=False, save_mode=SAVE_MODE, spike_fmt=SPIKE_FMT)
        snn.lif_backward(gs[i % 2], f, return_grad_v_init=False)
    torch.cuda.synchronize()
    torch.cuda._sleep(int(3e6 + 2.5e5 * reps))   # keep the GPU busy while the host enqueues
    for i in range(reps):
        e = ev[i]
        e[0].record(st)
        f = snn.lif_forward(xs[i % 2], p, return_v_final=False, save_mode=SAVE_MODE, spike_fmt=SPIKE_FMT)
        e[1].record(st)
        e[2].record(st)
        snn.lif_backward(gs[i % 2], f, return_grad_v_init=False)
        e[3].record(st)
    torch.cuda.synchronize()
    tf = sorted(e[0].elapsed_time(e[1]) for e in ev)[reps // 2]
    tb = sorted(e[2].elapsed_time(e[3]) for e in ev)[reps // 2]
    bf, bb = alg_bytes(dt, T, N)
    print(f"{dt:5s} T={T:4d} N={N:9d}{f' view+{off}' if off else ''}  fwd {tf * 1e3:8.1f} us {bf / tf / 1e6:7.0f} GB/s   "
          f"bwd {tb * 1e3:8.1f} us {bb / tb / 1e6:7.0f} GB/s", flush=True)
    return tf, tb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cases", default="cfg1,cfg2,t16")
    ap.add_argument("--save-mode", default="recompute")
    ap.add_argument("--spike-fmt", default="u8")
    a = ap.parse_args()
    global SAVE_MODE, SPIKE_FMT
    SAVE_MODE = a.save_mode
    SPIKE_FMT = a.spike_fmt
    torch.cuda.set_device(0)
    time_null(a.reps)
    for c in a.cases.split(","):
        for case in CASES[c]:
            time_case(*case[:3], a.reps, *case[3:])


if __name__ == "__main__":
    main()
