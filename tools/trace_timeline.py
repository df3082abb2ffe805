"""Per-CTA timeline of the TMA kernels (diagnostic; needs the -DSNN_TRACE library built by
tools/variant_build.py --name trace -DSNN_TRACE).  For each launch: when its first CTA entered, when griddepcontrol.wait
released, when the first ring stage landed, when the last CTA exited, CTAs / tiles, and the
gap to the previous launch -- the fixed per-launch costs that bound small layers.

    python tools/trace_timeline.py [--scenario cfg2|t8|t8flush|t32] [--reps 3]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SNN_LIF_LIBRARY", os.path.join(ROOT, "paper_2408_00280_b200", "build_trace",
                                                      "libsnn_lif_trace.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402
from paper_2408_00280_b200 import _lib  # noqa: E402
import snn_synth  # noqa: E402

REC = np.dtype([("kind", "<u4"), ("grid", "<u4"), ("smid", "<u4"), ("tiles", "<u4"), ("T", "<i8"), ("N", "<i8"),
                ("t_entry", "<u8"), ("t_wait", "<u8"), ("t_first", "<u8"), ("t_end", "<u8"),
                ("first_stolen", "<i4"), ("last_tile", "<i4"), ("t_issue", "<u8")])
KIND = {1: "fwd", 2: "bwd", 3: "bwdH"}
ORDER = False


def read_trace():
    n_max = 1 << 16
    buf = np.zeros(n_max, dtype=REC)
    f = _lib.lib.snn_trace_read
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    f.restype = ctypes.c_int
    n = f(buf.ctypes.data, n_max)
    assert n >= 0, "snn_trace_read failed (not a -DSNN_TRACE build?)"
    return buf[:n]


def report(recs, title):
    print(f"== {title}: {len(recs)} CTA records")
    if len(recs) == 0:
        return
    recs = np.sort(recs, order="t_entry")
    # split into launches: same (kind, grid, T, N) and overlapping in time with the group
    launches = []
    for r in recs:
        key = (int(r["kind"]), int(r["grid"]), int(r["T"]), int(r["N"]))
        for L in reversed(launches[-4:]):
            if L["key"] == key and r["t_entry"] <= L["end"] + 500 and L["n"] < key[1]:
                L["rows"].append(r); L["n"] += 1; L["end"] = max(L["end"], int(r["t_end"]))
                break
        else:
            launches.append(dict(key=key, rows=[r], n=1, end=int(r["t_end"])))
    t0 = int(recs["t_entry"].min())
    prev_end = None
    print(f"{'launch':>22} {'ctas':>5} {'tiles':>6} {'entry':>8} {'wait0':>8} {'wait1':>8} {'first0':>8} "
          f"{'first_med':>9} {'end_med':>8} {'end':>8} {'dur':>7} {'gap':>6} {'GB/s':>6} {'issue_med':>9} "
          f"[us, from the first entry; GB/s = alg. bytes / (end - wait0); issue = producer's first loads]")
    for L in launches:
        a = np.array(L["rows"], dtype=REC)
        k, grid, T, N = L["key"]
        us = lambda v: (int(v) - t0) / 1e3
        ent = a["t_entry"].min(); end = a["t_end"].max()
        gap = "  --  " if prev_end is None else f"{(int(ent) - prev_end) / 1e3:6.2f}"
        esz = 2 if k_is_bf16(T, N) else 4
        ck = 4.0 * (-(-T // 16) - 1) / T   # checkpoint rows after the first (V[-1] is not stored)
        nbytes = ((esz + 1 + ck) if k == 1 else (3 * esz + ck)) * T * N
        gbs = nbytes / max(1, int(end) - int(a["t_wait"].min()))
        print(f"{KIND.get(k, k):>5} T={T:<4d} N={N:<9d} {len(a):5d} {int(a['tiles'].sum()):6d} {us(ent):8.2f} "
              f"{us(a['t_wait'].min()):8.2f} {us(a['t_wait'].max()):8.2f} {us(a['t_first'].min()):8.2f} "
              f"{us(np.median(a['t_first'])):9.2f} {us(np.median(a['t_end'])):8.2f} {us(end):8.2f} "
              f"{(int(end) - int(ent)) / 1e3:7.2f} {gap} {gbs:6.0f} {us(np.median(a['t_issue'])):9.2f}")
        prev_end = int(end)
        if ORDER and grid > len(a):
            # steal order: first stolen tile of each CTA (sorted by time it was taken ~ entry order),
            # and the tiles that finished last
            fs = np.sort(a["first_stolen"][a["first_stolen"] >= 0])
            late = a[np.argsort(a["t_end"])[-8:]]
            print(f"        first stolen tiles: min {fs.min() if len(fs) else -1} max {fs.max() if len(fs) else -1}; "
                  f"last 8 CTAs to end ran tiles {list(late['last_tile'])} (grid {grid})")


def k_is_bf16(T, N):
    return T == 16 and N in cfg2_layers()


def cfg2_layers():
    B = 128
    return [B * 64 * 32 * 32, B * 128 * 16 * 16, B * 256 * 8 * 8, B * 256 * 8 * 8, B * 512 * 4 * 4,
            B * 512 * 4 * 4, B * 512 * 2 * 2, B * 512 * 2 * 2]


def scenario(name, reps):
    p = snn.LIFParams.paper()
    if name == "cfg2":
        specs = [(16, n, torch.bfloat16) for n in cfg2_layers()]
    elif name in ("t8", "t8flush"):
        specs = [(8, 1 << 20, torch.float32)]
    elif name in ("t32", "t128", "t512"):
        specs = [(int(name[1:]), 1 << 20, torch.float32)]
    else:
        raise SystemExit(f"unknown scenario {name}")
    bufs = []
    for T, N, dt in specs:
        XX = [snn_synth.normal_tensor(1234 + i, T, N, device="cuda", dtype=dt) for i in range(2)]
        GG = [snn_synth.normal_tensor(4321 + i, T, N, device="cuda", dtype=dt) for i in range(2)]
        ff = [snn.lif_forward(XX[i], p, return_v_final=False) for i in range(2)]
        bufs.append((XX, GG, ff, torch.empty_like(XX[0])))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if name == "t8flush" else None

    def step(i):
        for XX, GG, ff, gx in bufs:
            if flush is not None:
                flush.zero_()
            snn.lif_forward(XX[i], p, spikes=ff[i].spikes, saved=ff[i].saved, return_v_final=False)
            if flush is not None:
                flush.zero_()
            snn.lif_backward(GG[1 - i], ff[1 - i], grad_x=gx, return_grad_v_init=False)

    for i in range(3):
        step(i % 2)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(0)
        step(1)
    g.replay()
    torch.cuda.synchronize()
    for r in range(reps):
        read_trace()   # reset
        g.replay()
        torch.cuda.synchronize()
        report(read_trace(), f"{name} rep {r} (graph of 2 steps)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenario", default="cfg2")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--order", action="store_true", help="also print which tiles were stolen first / ran last")
    a = ap.parse_args()
    global ORDER
    ORDER = a.order
    torch.cuda.set_device(0)
    for s in a.scenario.split(","):
        scenario(s, a.reps)


if __name__ == "__main__":
    main()
