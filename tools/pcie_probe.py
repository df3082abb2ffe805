"""PCIe ceiling for the e2e leg: pinned host <-> device copy bandwidth, each direction alone and
both at once on two streams (1 GiB buffers, CUDA events, best of 5).

    python tools/pcie_probe.py
"""
import torch


def main():
    n = 1 << 30
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    def h2d():
        d_in.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_out, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1); cur.wait_stream(s2)

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(f"H2D {n / t1 / 1e6:.1f} GB/s  D2H {n / t2 / 1e6:.1f} GB/s  both at once {2 * n / t3 / 1e6:.1f} GB/s "
          f"({t1:.2f} / {t2:.2f} / {t3:.2f} ms per GiB)")


if __name__ == "__main__":
    main()


def strided():
    """2-D (strided) vs 1-D copies of the e2e leg's chunk shape: 512 rows x 64 KB (a 16 K-neuron
    column chunk of a [512, 2^20] fp32 host tensor) against one contiguous 32 MiB copy."""
    T, N, nc = 512, 1 << 20, 16384
    h = torch.empty(T * N * 4, dtype=torch.uint8).pin_memory()
    d = torch.empty(T * nc * 4, dtype=torch.uint8, device="cuda")
    import ctypes
    cudart = ctypes.CDLL("libcudart.so.12")
    cudart.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                         ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    st = torch.cuda.current_stream()

    def c2d():
        for k in range(8):
            cudart.cudaMemcpy2DAsync(d.data_ptr(), nc * 4, h.data_ptr() + k * nc * 4, N * 4, nc * 4, T, 1,
                                     ctypes.c_void_p(st.cuda_stream))

    def c1d():
        for k in range(8):
            d.copy_(h[k * T * nc * 4:(k + 1) * T * nc * 4], non_blocking=True)
    for name, fn in (("2-D 512 x 64 KB", c2d), ("1-D 32 MiB", c1d)):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"H2D {name}: {8 * T * nc * 4 / best / 1e6:.1f} GB/s")


if __name__ == "__main__":
    strided()
