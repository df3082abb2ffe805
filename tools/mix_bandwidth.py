"""HBM bandwidth of plain torch kernels at the fused LIF kernels' read:write mixes (a
mix-matched reference beside MEASURED_PEAKS.json's copy figure): copy (1:1), add (2:1, the
backward's ~8 B read : 4 B write) and a read-only reduction.

    python tools/mix_bandwidth.py
"""
import torch


def bench(fn, nbytes, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in evs)[reps // 2]
    return nbytes / (t / 1e3) / 1e9


def main():
    n = 1 << 29   # 2 GiB of fp32 per tensor
    a, b, e = (torch.empty(n, device="cuda").normal_() for _ in range(3))
    print(f"copy 1:1      {bench(lambda: e.copy_(a), 8 * n):8.0f} GB/s")
    print(f"add  2:1      {bench(lambda: torch.add(a, b, out=e), 12 * n):8.0f} GB/s")
    print(f"read-only sum {bench(lambda: a.sum(), 4 * n):8.0f} GB/s")


if __name__ == "__main__":
    main()
