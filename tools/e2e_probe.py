"""Where the e2e leg's time goes (diagnostic): the host-buffer path's copy pattern at cfg1 (T=512,
N=2^20 fp32, 16 K-neuron column chunks) replayed with bare 2-D copies -- H2D only, D2H only, both
directions on two streams without kernels -- against snn_lif_fwd_bwd_host itself.

    python tools/e2e_probe.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_00280_b200 as snn  # noqa: E402

T, N, NC = 512, 1 << 20, 16384
cudart = ctypes.CDLL("libcudart.so.12")
cudart.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]


def main():
    p = snn.LIFParams.paper()
    X = torch.randn(T, N).pin_memory()
    G = torch.randn(T, N).pin_memory()
    S = torch.empty(T, N, dtype=torch.uint8).pin_memory()
    GX = torch.empty(T, N).pin_memory()
    d = [torch.empty(T * NC * 4, dtype=torch.uint8, device="cuda") for _ in range(4)]
    ds = torch.empty(T * NC, dtype=torch.uint8, device="cuda")
    sin, sout = torch.cuda.Stream(), torch.cuda.Stream()

    def cp(dst, dpitch, src, spitch, width, kind, stream):
        assert cudart.cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, T, kind,
                                        ctypes.c_void_p(stream.cuda_stream)) == 0

    def h2d():
        for c in range(N // NC):
            cp(d[0].data_ptr(), NC * 4, X.data_ptr() + c * NC * 4, N * 4, NC * 4, 1, sin)
            cp(d[1].data_ptr(), NC * 4, G.data_ptr() + c * NC * 4, N * 4, NC * 4, 1, sin)

    def d2h():
        for c in range(N // NC):
            cp(S.data_ptr() + c * NC, N, ds.data_ptr(), NC, NC, 2, sout)
            cp(GX.data_ptr() + c * NC * 4, N * 4, d[2].data_ptr(), NC * 4, NC * 4, 2, sout)

    def both():
        h2d()
        d2h()

    ws = snn.host_workspace(T, N, p)

    def api():
        snn.lif_fwd_bwd_host(X, G, p, spikes=S, grad_x=GX, workspace=ws)

    for name, fn in (("H2D only (x, gS: 4.29 GB)", h2d), ("D2H only (spikes, gX: 2.68 GB)", d2h),
                     ("both, two streams, no kernels", both), ("snn_lif_fwd_bwd_host", api)):
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            sin.synchronize(); sout.synchronize()
            torch.cuda.current_stream().wait_stream(sin)
            torch.cuda.current_stream().wait_stream(sout)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{name}: {best:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
