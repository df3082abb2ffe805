"""Small-T isolated-launch probe (tuning aid, not the bench contract).

For cfg1 shapes at small T, times each forward / backward launch alone (CUDA events, the
launches captured in one graph like bench.py --sweep) under three L2 preparations:

  dirty  -- a 512 MiB memset before every launch (bench.py --sweep's flush): L2 is left full
            of the memset's dirty lines, which the timed launch must write back as it evicts;
  clean  -- the same memset, then a 256 MiB read (a sum) so L2 holds clean lines only: a
            cold launch that pays nothing for its predecessor's write-backs;
  none   -- no flush; two input batches alternate (working set 2x the layer).

and for two kernel families: the TMA kernels (default) and the generic register-prefetch
kernels (SNN_LIF_NO_TMA=1, read by the library on every call).

    python tools/small_t_probe.py [--T 8,16,32] [--reps 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
import snn_synth  # noqa: E402


def run(T, N, prep, family, reps, dev):
    os.environ["SNN_LIF_NO_TMA"] = "1" if family == "generic" else "0"
    p = snn.LIFParams.paper()
    xs = [snn_synth.normal_tensor(1234 + i, T, N, device=dev) for i in range(2)]
    gs = [snn_synth.normal_tensor(4321 + i, T, N, device=dev) for i in range(2)]
    fs = [snn.lif_forward(xs[i], p, save_mode="recompute", return_v_final=False) for i in range(2)]
    gxs = [snn.lif_backward(gs[i], fs[i], return_grad_v_init=False)[0] for i in range(2)]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    rd = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    acc = torch.zeros((), dtype=torch.float32, device=dev)
    evs = []

    def prepare():
        if prep in ("dirty", "clean"):
            flush.zero_()
        if prep == "clean":
            torch.sum(rd, 0, out=acc)

    def one(i, record):
        b = i % 2
        e = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)] if record else None
        prepare()
        if record: e[0].record()
        snn.lif_forward(xs[b], p, save_mode="recompute", spikes=fs[b].spikes, saved=fs[b].saved,
                        return_v_final=False)
        if record: e[1].record()
        prepare()
        if record: e[2].record()
        snn.lif_backward(gs[b], fs[b], grad_x=gxs[b], return_grad_v_init=False)
        if record:
            e[3].record(); evs.append(e)

    for i in range(4):
        one(i, False)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            one(i, True)
    g.replay()
    torch.cuda.synchronize(dev)
    tf = sorted(e[0].elapsed_time(e[1]) for e in evs)[reps // 2]
    tb = sorted(e[2].elapsed_time(e[3]) for e in evs)[reps // 2]
    ck = 4.0 * (-(-T // 16) - 1) / T   # checkpoint rows after the first (V[-1] is not stored)
    bf, bb = (4 + 1 + ck) * T * N, (12 + ck) * T * N
    print(f"T={T:4d} N={N} {prep:5s} {family:7s} fwd {tf * 1e3:7.2f} us {bf / tf / 1e6:6.0f} GB/s  "
          f"bwd {tb * 1e3:7.2f} us {bb / tb / 1e6:6.0f} GB/s  fwd+bwd {(bf + bb) / (tf + tb) / 1e6:6.0f} GB/s "
          f"{T * N / ((tf + tb) / 1e3):.3e} ns/s", flush=True)
    os.environ["SNN_LIF_NO_TMA"] = "0"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", default="8,16,32")
    ap.add_argument("--N", type=int, default=1 << 20)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--preps", default="dirty,clean,none")
    ap.add_argument("--families", default="tma,generic")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    for T in [int(t) for t in a.T.split(",")]:
        for prep in a.preps.split(","):
            for fam in a.families.split(","):
                run(T, a.N, prep, fam, a.reps, dev)


if __name__ == "__main__":
    main()
