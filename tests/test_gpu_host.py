"""snn_lif_fwd_bwd_host (host-buffer runtime): chunked, stream-overlapped fwd+bwd over host
tensors must equal the device calls bitwise, for every chunking / slot count / format."""
import os
import sys

import pytest
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

pytestmark = pytest.mark.gpu

import paper_2408_00280_b200 as snn  # noqa: E402
import snn_synth  # noqa: E402

PAPER = snn.LIFParams.paper()


def _device_ref(X, G, p, spike_fmt, save_mode):
    f = snn.lif_forward(X.cuda(), p, spike_fmt=spike_fmt, save_mode=save_mode)
    gx, _ = snn.lif_backward(G.cuda(), f)
    torch.cuda.synchronize()
    return f.spikes.cpu(), gx.cpu()


@pytest.mark.parametrize("T,N,chunk,nslots,spike_fmt,save_mode,dtype", [
    (16, 5000, 512, 2, "u8", "recompute", torch.float32),      # 10 chunks, ragged last, 2 slots
    (37, 4096, 1024, 3, "bits", "recompute", torch.float32),
    (20, 3000, 512, 4, "io", "h", torch.float32),
    (16, 6000, 1536, 3, "u8", "recompute", torch.bfloat16),
    (8, 700, 0, 0, "u8", "recompute", torch.float32),           # defaults: one chunk
    (1, 1, 0, 0, "io", "recompute", torch.float32),             # degenerate
])
def test_host_path_equals_device_path_bitwise(T, N, chunk, nslots, spike_fmt, save_mode, dtype):
    X = snn_synth.normal_tensor(71, T, N, dtype=dtype).pin_memory()
    G = snn_synth.normal_tensor(72, T, N, dtype=dtype).pin_memory()
    s_ref, gx_ref = _device_ref(X, G, PAPER, spike_fmt, save_mode)
    S, GX = snn.lif_fwd_bwd_host(X, G, PAPER, spike_fmt=spike_fmt, save_mode=save_mode,
                                 chunk_neurons=chunk, nslots=nslots)
    assert torch.equal(S, s_ref)
    assert torch.equal(GX, gx_ref)


def test_host_path_strided_rows_and_pageable_memory():
    """Host rows with ld > N (a column view of a wider host tensor), not pinned."""
    T, N, ld = 12, 2000, 2600
    full_x = snn_synth.normal_tensor(73, T, ld)
    full_g = snn_synth.normal_tensor(74, T, ld)
    X, G = full_x[:, :N], full_g[:, :N]
    s_ref, gx_ref = _device_ref(X.contiguous(), G.contiguous(), PAPER, "u8", "recompute")
    S, GX = snn.lif_fwd_bwd_host(X, G, PAPER, chunk_neurons=512, nslots=3)
    assert torch.equal(S, s_ref) and torch.equal(GX, gx_ref)


def test_host_path_reuses_workspace_and_rejects_small_one():
    T, N = 8, 4096
    X = snn_synth.normal_tensor(75, T, N).pin_memory()
    G = snn_synth.normal_tensor(76, T, N).pin_memory()
    ws = snn.host_workspace(T, N, PAPER, chunk_neurons=1024, nslots=2)
    a = snn.lif_fwd_bwd_host(X, G, PAPER, chunk_neurons=1024, nslots=2, workspace=ws)
    b = snn.lif_fwd_bwd_host(X, G, PAPER, chunk_neurons=1024, nslots=2, workspace=ws)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    from paper_2408_00280_b200 import _lib
    from paper_2408_00280_b200.lif import make_shape
    shape = make_shape(X, "u8", "recompute")
    with pytest.raises(_lib.SNNError, match="workspace too small"):
        _lib.snn_lif_fwd_bwd_host(PAPER.to_c(), shape, X.data_ptr(), G.data_ptr(), a[0].data_ptr(),
                                  a[1].data_ptr(), 1024, 2, ws.data_ptr(), 1024, None)
