"""GPU: the RECOMPUTE checkpoint of V[-1] is not stored (r2c).

The forward checkpoints the V entering every 16-step chunk except the first: that one is
v_init (or V_reset), which snn_lif_backward receives itself (include/snn_lif.h; DESIGN.md
section 6).  For T <= 16 nothing is checkpointed at all.  These tests pre-fill the saved
buffer with NaN, so a kernel that still reads (or forgets to write) a checkpoint row would
poison the gradients, and compare with the oracle (Eq. 3) on both kernel
families.  The affine pair re-reads V[-1] the same way (a non-trivial v_init below); only
the handoff pair keeps storing it (it arrives inside the kernel; test_gpu_handoff.py).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_00280_b200 as snn  # noqa: E402
from paper_2408_00280_b200 import lif as L  # noqa: E402
import oracle  # noqa: E402
import snn_synth  # noqa: E402
from parity import compare, oracle_run  # noqa: E402

PAPER = snn.LIFParams.paper()
CFG0 = snn.LIFParams.north_star()


def _case(params, T, N, dtype, with_v0, seed):
    X = snn_synth.normal_tensor(seed, T, N, dtype=dtype)
    G = snn_synth.normal_tensor(seed + 1, T, N, dtype=dtype)
    v0 = snn_synth.normal_tensor(seed + 2, 1, N, std=0.5)[0] if with_v0 else None
    return X, G, v0


@pytest.mark.parametrize("family", ["tma", "generic"])
@pytest.mark.parametrize("T", [1, 8, 16, 17, 33, 48])
@pytest.mark.parametrize("with_v0", [False, True])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_nan_prefilled_saved_matches_oracle(family, T, with_v0, dtype, monkeypatch):
    monkeypatch.setenv("SNN_LIF_NO_TMA", "1" if family == "generic" else "0")
    N = 3000 if dtype == torch.float32 else 3072   # several tiles, a ragged last tile
    p = PAPER if T % 2 else CFG0
    X, G, v0 = _case(p, T, N, dtype, with_v0, 700 + T)
    xd, gd = X.cuda(), G.cuda()
    shape = L.make_shape(xd, "u8", "recompute")
    saved = torch.full((L.saved_bytes(p, shape) // 4,), float("nan"), device="cuda")
    f = snn.lif_forward(xd, p, v_init=None if v0 is None else v0.cuda(), saved=saved)
    gx, gvi = snn.lif_backward(gd, f)
    torch.cuda.synchronize()
    ref = oracle_run(p, X, G, v0, None)
    rep = compare(p, ref, ref["gX"], ref["gvi"], f.spikes.cpu(), gx.cpu(), vf_gpu=f.v_final.cpu(),
                  gvi_gpu=gvi.cpu(), io_bf16=(dtype == torch.bfloat16))
    assert rep.ok, str(rep)
    ck = saved.view(-1, (N + 15) // 16 * 16)   # [ceil(T/16), round_up(N, 16)] (snn_lif_api.cu saved_ld)
    assert torch.isnan(ck[0, :N]).all(), "checkpoint row 0 (V[-1]) was written"
    if T > 16:
        assert not torch.isnan(ck[1:(T + 15) // 16, :N]).any()


def test_backward_reads_v_init():
    """The backward's V[-1] is its own v_init argument: the same forward state with another
    v_init gives other gradients (the contract in include/snn_lif.h), the right one the
    oracle's."""
    T, N = 12, 2048
    X, G, v0 = _case(PAPER, T, N, torch.float32, True, 811)
    xd, gd, v0d = X.cuda(), G.cuda(), v0.cuda()
    f = snn.lif_forward(xd, PAPER, v_init=v0d)
    gx, _ = snn.lif_backward(gd, f)
    wrong = L.LIFForward(f.spikes, f.saved, f.v_final, xd, None, PAPER, f.shape)
    gx_wrong, _ = snn.lif_backward(gd, wrong)
    torch.cuda.synchronize()
    assert not torch.equal(gx, gx_wrong)
    ref = oracle_run(PAPER, X, G, v0, None)
    rep = compare(PAPER, ref, ref["gX"], ref["gvi"], f.spikes.cpu(), gx.cpu(), vf_gpu=f.v_final.cpu())
    assert rep.ok, str(rep)


@pytest.mark.parametrize("family", ["tma", "generic"])
@pytest.mark.parametrize("T", [8, 40])
def test_affine_pair_v_init(family, T, monkeypatch):
    """snn_lif_backward_affine re-reads V[-1] from its v_init like snn_lif_backward: a
    non-trivial v_init through the affine pair matches the oracle."""
    monkeypatch.setenv("SNN_LIF_NO_TMA", "1" if family == "generic" else "0")
    B, C, HW = 4, 8, 64
    N = B * C * HW
    X, G, v0 = _case(PAPER, T, N, torch.float32, True, 900 + T)
    gen = torch.Generator().manual_seed(T)
    sc = torch.rand(C, generator=gen) + 0.5
    sh = 0.2 * torch.randn(C, generator=gen)
    af = snn.AffineSpec(sc.cuda(), sh.cuda(), C, HW)
    f = snn.lif_forward_affine(X.cuda(), PAPER, af, v_init=v0.cuda())
    gx, gvi, _, _ = snn.lif_backward_affine(G.cuda(), f)
    torch.cuda.synchronize()
    Xp = oracle.affine_input(X.double().numpy(), sc.double().numpy(), sh.double().numpy(), C, HW)
    ref = oracle_run(PAPER, Xp, G, v0, None)
    rgx, _, _ = oracle.affine_grads(X.double().numpy(), ref["gX"], sc.double().numpy(), C, HW)
    cidx = (np.arange(N) // HW) % C
    ref_scaled = dict(ref)
    ref_scaled["gX_bound"] = ref["gX_bound"] * np.abs(sc.double().numpy())[cidx][None, :]
    rep = compare(PAPER, ref_scaled, rgx, ref["gvi"], f.spikes.cpu(), gx.cpu(), vf_gpu=f.v_final.cpu(),
                  gvi_gpu=gvi.cpu())
    assert rep.ok, str(rep)
