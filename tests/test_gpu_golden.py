"""The hand-derived golden traces (tests/golden/, each value cited there) run through the CUDA
kernels.  Dyadic forward values (H, S, V) must come out of the kernels bit for bit in fp32;
the non-dyadic backward values (SPEC / hand traces in fp64 decimals) within the fp32 +
MUFU-approximation error (a few ulp).  Exact threshold ties (p15) MUST fire: Eq. 2's ">="
 -- the parity comparator's tie rule is not applied here, so a kernel
that compared with ">" fails.  Every trace runs on both kernel families: N = 1 (the generic
kernels) and the trace replicated over N = 1024 aligned columns (the TMA kernels)."""
import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_00280_b200 as snn  # noqa: E402

CFG0 = snn.LIFParams.north_star()           # tau=2, V_th=1, V_reset=0, hard, decay_input
PAPER = snn.LIFParams.paper()               # tau=1.25, V_th=0.3, V_rest=0, Eq. 1
f32 = lambda v: np.float32(v)


def trace(params, xs, N, *, dtype=torch.float32, gs=None, gvf=None, save_mode="h"):
    """Run the trace xs[t] (same value in every column) through lif_forward / lif_backward.
    Returns per-step H (save_mode h), S, V (V[t] = v_final of the prefix run 0..t), gX, gvi
    of column 0, after checking every column agrees bitwise."""
    T = len(xs)
    X = torch.tensor(xs, dtype=torch.float32).to(dtype).view(T, 1).repeat(1, N).cuda()
    f = snn.lif_forward(X, params, save_mode=save_mode)
    torch.cuda.synchronize()
    S = f.spikes.cpu().numpy().astype(np.float64)
    assert (S == S[:, :1]).all()
    H = None
    if save_mode == "h":
        ldh = (N + 15) // 16 * 16
        Hm = f.saved.view(T, ldh)[:, :N].cpu().numpy()
        assert (Hm == Hm[:, :1]).all()
        H = Hm[:, 0]
    V = []
    for t in range(T):
        ft = snn.lif_forward(X[: t + 1].contiguous(), params, save_mode="none")
        V.append(ft.v_final[0].item())
    out = dict(H=H, S=S[:, 0], V=np.array(V, dtype=np.float32))
    if gs is not None:
        G = torch.tensor(gs, dtype=torch.float32).to(dtype).view(T, 1).repeat(1, N).cuda()
        g_in = None if gvf is None else torch.full((N,), float(gvf), device="cuda")
        gx, gvi = snn.lif_backward(G, f, grad_v_final=g_in)
        torch.cuda.synchronize()
        gxn = gx.float().cpu().numpy()
        assert (gxn == gxn[:, :1]).all()
        out["gX"] = gxn[:, 0].astype(np.float64)
        out["gvi"] = float(gvi[0].item())
    return out


NS = [1, 1024]   # generic kernels, TMA kernels


@pytest.mark.parametrize("N", NS)
@pytest.mark.parametrize("save_mode", ["h", "recompute"])
def test_p1_constant_current_cfg0_bitwise(N, save_mode):
    g = load_golden("p1_constant_current.txt")
    r = trace(CFG0, [1.5] * 8, N, save_mode=save_mode)
    if save_mode == "h":
        assert r["H"].tolist() == g["cfg0_x1p5_H"]          # dyadic: exact in fp32
    assert r["S"].tolist() == g["cfg0_x1p5_S"]
    assert r["V"].tolist() == g["cfg0_x1p5_V"]
    assert trace(CFG0, [1.2] * 8, N, save_mode=save_mode)["S"].tolist() == g["cfg0_x1p2_S"]


@pytest.mark.parametrize("N", NS)
def test_p1_constant_current_paper(N):
    g = load_golden("p1_constant_current.txt")
    r = trace(PAPER, [0.26] * 6, N)
    assert r["S"].tolist() == g["paper_x0p26_S"]
    assert r["H"][0] == f32(g["paper_x0p26_H01"][0])                       # H[0] = x exactly
    np.testing.assert_allclose(r["H"][1], g["paper_x0p26_H01"][1], rtol=2e-7)  # fma(k, x, x)
    assert trace(PAPER, [0.5] * 4, N)["S"].tolist() == g["paper_x0p5_S"]


@pytest.mark.parametrize("N", NS)
def test_p3_spec_reset_example_bitwise(N):
    g = load_golden("p3_spec_reset.txt")
    r = trace(PAPER, g["x"], N)
    assert r["H"].tolist() == [f32(v) for v in g["H"]]
    assert r["S"].tolist() == g["S"]
    assert r["V"].tolist() == [f32(v) for v in g["V"]]


@pytest.mark.parametrize("N", NS)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_p4_soft_reset_dyadic_bitwise(N, dtype):
    g = load_golden("p4_soft_reset.txt")
    r = trace(snn.LIFParams.north_star(reset="soft"), [1.5] * 6, N, dtype=dtype)
    assert r["H"].tolist() == g["H"] and r["S"].tolist() == g["S"] and r["V"].tolist() == g["V"]


@pytest.mark.parametrize("N", NS)
@pytest.mark.parametrize("save_mode", ["h", "recompute"])
def test_p15_exact_ties_fire(N, save_mode):
    """H == V_th exactly spikes (Eq. 2 '>='); no tie excuse."""
    g = load_golden("p15_exact_ties.txt")
    r = trace(CFG0, [2.0] * 4, N, save_mode=save_mode)
    assert r["S"].tolist() == g["cfg0_x2_S"]
    if save_mode == "h":
        assert r["H"].tolist() == g["cfg0_x2_H"]
    r = trace(CFG0, [1.0] * 4, N, save_mode=save_mode)
    assert r["S"].tolist() == g["cfg0_x1_S"]
    if save_mode == "h":
        assert r["H"].tolist() == g["cfg0_x1_H"]
    assert trace(PAPER, [0.3] * 3, N, save_mode=save_mode)["S"].tolist() == g["paper_x0p3_S"]
    assert trace(PAPER, [0.3, 0.0, 0.0], N, save_mode=save_mode)["S"].tolist() == g["paper_x0p3_then0_S"]


@pytest.mark.parametrize("N", NS)
@pytest.mark.parametrize("save_mode", ["h", "recompute"])
def test_p6_spec_backward_examples(N, save_mode):
    g = load_golden("p6_spec_backward.txt")
    # (b) g_y = 1 at v = V_th (u = 0), y = 1: g_x = delta(0) = alpha / 4 = 1.0
    r = trace(PAPER, [0.3], N, gs=[1.0], save_mode=save_mode)
    assert r["S"].tolist() == [1.0]
    np.testing.assert_allclose(r["gX"][0], g["b_gx"][0], rtol=1e-6)
    # (c) g_v_next = 1, g_y = 0, v = 0.1, y = 0: g_x = 0.2 (1 - 0.1 delta(-0.2))
    r = trace(PAPER, g["c_x"], N, gs=[0.0], gvf=g["c_grad_v_final"][0], save_mode=save_mode)
    assert r["S"].tolist() == [0.0]
    np.testing.assert_allclose(r["gX"][0], g["c_gx"][0], rtol=2e-6)
    # (a) zero in, zero out
    r = trace(PAPER, [0.1], N, gs=[0.0], save_mode=save_mode)
    assert r["gX"][0] == 0.0


@pytest.mark.parametrize("N", NS)
@pytest.mark.parametrize("save_mode", ["h", "recompute"])
def test_p7_two_step_backward(N, save_mode):
    g = load_golden("p7_backward_two_step.txt")
    r = trace(CFG0, [1.5, 1.5], N, gs=[1.0, 1.0], save_mode=save_mode)
    assert r["S"].tolist() == [0.0, 1.0]
    np.testing.assert_allclose(r["gX"], g["gX"], rtol=2e-6)
    np.testing.assert_allclose(r["gvi"], g["grad_v_init"][0], rtol=2e-6)
    r = trace(snn.LIFParams.north_star(detach_reset=True), [1.5, 1.5], N, gs=[1.0, 1.0], save_mode=save_mode)
    np.testing.assert_allclose(r["gX"], g["gX_detach"], rtol=2e-6)
    np.testing.assert_allclose(r["gvi"], g["grad_v_init_detach"][0], rtol=2e-6)


@pytest.mark.parametrize("N", [5, 1024])   # ragged N: generic kernels; 1024: TMA kernels
def test_infinities_propagate_like_the_oracle(N):
    """+-Inf currents, paper mode (Eq. 1's k v + x): +Inf fires and hard-resets to
    V_reset, -Inf stays silent and leaves V = -Inf for good; the oracle on the same input agrees
    on every spike, H, V and gradient (NaN where (V_reset - H) delta is Inf * 0, on both sides)."""
    from parity import compare, oracle_run
    T = 6
    cols = [[0.4, float("inf"), 0.1, 0.2, 0.5, 0.1],
            [0.2, float("-inf"), 0.4, 0.1, 0.2, 0.3],
            [float("inf")] * T,
            [0.1, 0.2, 0.1, 0.2, float("-inf"), 0.9]]
    X = torch.tensor(cols, dtype=torch.float32).t().contiguous()       # [T, 4]
    X = X.repeat(1, -(-N // 4))[:, :N].contiguous()
    G = torch.linspace(-1, 1, T * X.shape[1]).view(T, -1).contiguous()
    f = snn.lif_forward(X.cuda(), PAPER, save_mode="h")
    gx, gvi = snn.lif_backward(G.cuda(), f)
    torch.cuda.synchronize()
    ref = oracle_run(PAPER, X, G)
    ldh = (X.shape[1] + 15) // 16 * 16
    rep = compare(PAPER, ref, ref["gX"], ref["gvi"], f.spikes.cpu(), gx.cpu(),
                  H_gpu=f.saved.view(T, ldh)[:, : X.shape[1]].cpu(), vf_gpu=f.v_final.cpu(), gvi_gpu=gvi.cpu())
    assert rep.ok, str(rep)
    S = f.spikes.cpu().numpy()
    assert S[1, 0] == 1 and S[1, 1] == 0 and S[:, 2].tolist() == [1] * T
    vf = f.v_final.cpu().numpy()
    assert np.isneginf(vf[1]) and np.isneginf(vf[3]) and vf[2] == 0.0
    assert np.isnan(gx.cpu().numpy()[1, 0]) and np.isnan(ref["gX"][1, 0])   # (0 - Inf) * 0 on both sides
