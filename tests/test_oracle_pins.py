"""Pins for the CPU oracle.

Every check here compares the oracle with something other than itself: the paper's or
SPEC's worked examples and exact hand traces (tests/golden/), closed forms, scipy
library routines (lfilter, expit, quad), the paper's literal Eq. 1 / Eq. 3 recursions at
V_reset = 0, invariants, and finite differences of the surrogate-smoothed model.
"""
import math

import numpy as np
import pytest
from scipy import integrate, signal, special

from conftest import load_golden
from oracle import OracleParams, backward, forward, smooth_step, surrogate

CFG0 = OracleParams(tau=2.0, v_th=1.0, v_reset=0.0, decay_input=True)     # BJ.configs[0]
PAPER = OracleParams(tau=1.25, v_th=0.3, v_reset=0.0, decay_input=False)


def col(v, T):
    return np.full((T, 1), v, dtype=np.float64)


# ----------------------------------------------------------------------------- P1

def test_p1_constant_current_cfg0_golden():
    g = load_golden("p1_constant_current.txt")
    r = forward(CFG0, col(1.5, 8))
    assert r["H"][:, 0].tolist() == g["cfg0_x1p5_H"]
    assert r["S"][:, 0].tolist() == g["cfg0_x1p5_S"]
    assert r["V"][:, 0].tolist() == g["cfg0_x1p5_V"]
    r = forward(CFG0, col(1.2, 8))
    assert r["S"][:, 0].tolist() == g["cfg0_x1p2_S"]


def test_p1_constant_current_paper_golden():
    g = load_golden("p1_constant_current.txt")
    r = forward(PAPER, col(0.26, 6))
    np.testing.assert_allclose(r["H"][:2, 0], g["paper_x0p26_H01"], rtol=1e-15)
    assert r["S"][:, 0].tolist() == g["paper_x0p26_S"]
    assert forward(PAPER, col(0.5, 4))["S"][:, 0].tolist() == g["paper_x0p5_S"]


def test_p15_exact_ties_fire():
    """Eq. 2's ">=": H == V_th exactly must spike (tests/golden/p15)."""
    g = load_golden("p15_exact_ties.txt")
    r = forward(CFG0, col(2.0, 4))
    assert r["H"][:, 0].tolist() == g["cfg0_x2_H"] and r["S"][:, 0].tolist() == g["cfg0_x2_S"]
    r = forward(CFG0, col(1.0, 4))
    assert r["H"][:, 0].tolist() == g["cfg0_x1_H"] and r["S"][:, 0].tolist() == g["cfg0_x1_S"]
    f32 = lambda v: float(np.float32(v))
    p = OracleParams(tau=f32(1.25), v_th=f32(0.3), v_reset=0.0)   # the fp32 values a kernel gets
    assert forward(p, col(f32(0.3), 3))["S"][:, 0].tolist() == g["paper_x0p3_S"]
    x = np.array([[f32(0.3)], [0.0], [0.0]])
    assert forward(p, x)["S"][:, 0].tolist() == g["paper_x0p3_then0_S"]


@pytest.mark.parametrize("X", [1.07, 1.3, 1.61, 2.2, 3.9, 7.3])
@pytest.mark.parametrize("tau", [1.5, 2.0, 4.0])
def test_p1_closed_form_period_decay_input(X, tau):
    """decay_input=1, V_reset=0, v_init=0: H[t] = X(1 - k^{t+1}) until the first spike;
    hard reset restarts the orbit, so S has period P = ceil(ln(1 - V_th/X)/ln k)."""
    p = OracleParams(tau=tau, v_th=1.0, v_reset=0.0, decay_input=True)
    k = 1.0 - 1.0 / tau
    P = math.ceil(math.log(1.0 - 1.0 / X) / math.log(k))
    T = 6 * P + 3
    r = forward(p, col(X, T))
    t = np.arange(P)
    np.testing.assert_allclose(r["H"][:P, 0], X * (1.0 - k ** (t + 1)), rtol=1e-13)
    expected = np.array([1.0 if (i % P) == P - 1 else 0.0 for i in range(T)])
    np.testing.assert_array_equal(r["S"][:, 0], expected)


@pytest.mark.parametrize("x", [0.245, 0.27, 0.33, 0.61])
def test_p1_closed_form_period_paper_mode(x):
    """Paper Eq. 1 (decay_input=0): H[t] = x(1-k^{t+1})/(1-k) before the first spike,
    period P = ceil(ln(1 - V_th(1-k)/x)/ln k) for x > V_th(1-k)."""
    k = 1.0 - 1.0 / PAPER.tau
    P = max(1, math.ceil(math.log(1.0 - PAPER.v_th * (1 - k) / x) / math.log(k)))
    T = 5 * P + 2
    r = forward(PAPER, col(x, T))
    t = np.arange(P)
    np.testing.assert_allclose(r["H"][:P, 0], x * (1 - k ** (t + 1)) / (1 - k), rtol=1e-13)
    expected = np.array([1.0 if (i % P) == P - 1 else 0.0 for i in range(T)])
    np.testing.assert_array_equal(r["S"][:, 0], expected)


def test_p1_closed_form_with_v_reset_offset():
    """decay_input=1 with V_reset = r, v_init = r: the charge relaxes to X + r, so
    H[t] = (X + r) - X k^{t+1} before the first spike."""
    r0, X, tau = 0.25, 1.4, 2.0
    p = OracleParams(tau=tau, v_th=1.0, v_reset=r0, decay_input=True)
    k = 1 - 1 / tau
    out = forward(p, col(X, 3), v_init=np.array([r0]))
    t = np.arange(2)
    np.testing.assert_allclose(out["H"][:2, 0], (X + r0) - X * k ** (t + 1), rtol=1e-14)


# ----------------------------------------------------------------------------- P2

@pytest.mark.parametrize("decay_input", [True, False])
def test_p2_subthreshold_is_linear_iir(decay_input):
    """Sub-threshold input never spikes and H is the IIR lfilter([s], [1, -k], X)
    (scipy.signal.lfilter), including a non-zero initial state via zi."""
    rng = np.random.default_rng(7)
    tau = 2.0 if decay_input else 1.25
    v_th = 1.0 if decay_input else 0.3
    p = OracleParams(tau=tau, v_th=v_th, v_reset=0.0, decay_input=decay_input)
    k = 1 - 1 / tau
    s = 1 / tau if decay_input else 1.0
    # sup of the orbit = s X/(1-k) (+ k^{t+1} v0) must stay below V_th
    xmax = 0.9 * v_th * (1 - k) / s
    T, N = 20, 6
    X = rng.uniform(-xmax, xmax, size=(T, N))
    v0 = rng.uniform(-0.2, 0.2, size=N) * v_th
    r = forward(p, X, v_init=v0)
    assert r["S"].sum() == 0
    ref = np.stack([signal.lfilter([s], [1.0, -k], X[:, n], zi=[k * v0[n]])[0]
                    for n in range(N)], axis=1)
    np.testing.assert_allclose(r["H"], ref, rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(r["v_final"], ref[-1], rtol=1e-13)


def test_p2_cfg0_x0p9_never_spikes():
    r = forward(CFG0, col(0.9, 200))
    assert r["S"].sum() == 0
    assert r["H"][-1, 0] < 0.9


# ----------------------------------------------------------------------------- P3 / P4

def test_p3_spec_reset_example():
    g = load_golden("p3_spec_reset.txt")
    r = forward(PAPER, np.array(g["x"])[:, None])
    np.testing.assert_allclose(r["H"][:, 0], g["H"], rtol=1e-15)
    assert r["S"][:, 0].tolist() == g["S"]
    np.testing.assert_allclose(r["V"][:, 0], g["V"], rtol=1e-15)


def test_p4_soft_reset_dyadic_trace():
    g = load_golden("p4_soft_reset.txt")
    p = OracleParams(tau=2.0, v_th=1.0, v_reset=0.0, soft_reset=True, decay_input=True)
    r = forward(p, col(1.5, 6))
    assert r["H"][:, 0].tolist() == g["H"]
    assert r["S"][:, 0].tolist() == g["S"]
    assert r["V"][:, 0].tolist() == g["V"]


# ----------------------------------------------------------------------------- P5

@pytest.mark.parametrize("alpha", [1.0, 2.0, 4.0, 9.5])
def test_p5_sigmoid_surrogate_closed_forms(alpha):
    p = OracleParams(alpha=alpha, surrogate="sigmoid")
    assert surrogate(p, 0.0) == alpha / 4          # sigma'(0) = alpha/4
    for u in [0.01, 0.3, 1.7, 5.0]:
        # library routine: delta = alpha sigma(alpha u)(1 - sigma(alpha u)), scipy expit
        e = special.expit(alpha * u)
        assert surrogate(p, u) == pytest.approx(alpha * e * (1 - e), rel=1e-12)
        assert surrogate(p, u) == surrogate(p, -u)
        assert surrogate(p, u) < surrogate(p, 0.0)
    val, err = integrate.quad(lambda u: surrogate(p, u), -60 / alpha, 60 / alpha, limit=200)
    assert val == pytest.approx(1.0, abs=1e-9)


def test_p5_sigmoid_tail_value():
    p = OracleParams(alpha=4.0)
    d10 = surrogate(p, 10.0)
    assert d10 < 1e-16
    assert d10 == pytest.approx(4 * math.exp(-40), rel=1e-12)  # (1+e^-40)^2 == 1 in fp64


@pytest.mark.parametrize("alpha", [1.0, 2.0, 4.0])
def test_p5_atan_surrogate_closed_forms(alpha):
    p = OracleParams(alpha=alpha, surrogate="atan")
    assert surrogate(p, 0.0) == alpha / 2
    for u in [0.05, 0.4, 3.0]:
        assert surrogate(p, u) == surrogate(p, -u)
    # integral over R of (a/2)/(1+(pi a u/2)^2) is 1; quad over R directly
    val, _ = integrate.quad(lambda u: surrogate(p, u), -np.inf, np.inf)
    assert val == pytest.approx(1.0, abs=1e-9)


@pytest.mark.parametrize("kind", ["sigmoid", "atan"])
def test_p5_delta_is_derivative_of_smooth_step(kind):
    p = OracleParams(alpha=3.0, surrogate=kind)
    assert smooth_step(p, 0.0) == 0.5
    assert smooth_step(p, 5000.0) == pytest.approx(1.0, abs=1e-4)
    assert smooth_step(p, -5000.0) == pytest.approx(0.0, abs=1e-4)
    h = 1e-6
    for u in [-1.3, -0.2, 0.0, 0.07, 0.9]:
        fd = (smooth_step(p, u + h) - smooth_step(p, u - h)) / (2 * h)
        assert surrogate(p, u) == pytest.approx(fd, rel=1e-7, abs=1e-10)


# ----------------------------------------------------------------------------- P6 / P7

def test_p6_spec_backward_examples():
    g = load_golden("p6_spec_backward.txt")
    # (a) zero upstream -> zero gradient
    r = forward(PAPER, col(0.2, 3))
    gX, gvi = backward(PAPER, np.zeros((3, 1)), r["H"])
    assert np.all(gX == 0) and np.all(gvi == 0)
    # (b) at threshold: H = 0.3 exactly (x = 0.3 from rest), g_y = 1 -> delta(0) = 1
    r = forward(PAPER, col(0.3, 1))
    assert r["S"][0, 0] == 1.0 and r["H"][0, 0] == 0.3
    gX, _ = backward(PAPER, np.ones((1, 1)), r["H"])
    assert gX[0, 0] == g["b_gx"][0]
    # (c) g_v_next = 1, g_y = 0, v = 0.1, y = 0
    r = forward(PAPER, col(g["c_x"][0], 1))
    gX, _ = backward(PAPER, np.zeros((1, 1)), r["H"], grad_v_final=np.array(g["c_grad_v_final"]))
    assert gX[0, 0] == pytest.approx(g["c_gx"][0], rel=1e-14)


def test_p7_two_step_backward_hand_trace():
    g = load_golden("p7_backward_two_step.txt")
    r = forward(CFG0, col(1.5, 2))
    assert r["H"][:, 0].tolist() == [0.75, 1.125] and r["S"][:, 0].tolist() == [0, 1]
    gX, gvi = backward(CFG0, np.ones((2, 1)), r["H"])
    np.testing.assert_allclose(gX[:, 0], g["gX"], rtol=1e-14)
    np.testing.assert_allclose(gvi, g["grad_v_init"], rtol=1e-14)
    pd = OracleParams(tau=2.0, v_th=1.0, v_reset=0.0, decay_input=True, detach_reset=True)
    gX, gvi = backward(pd, np.ones((2, 1)), r["H"])
    np.testing.assert_allclose(gX[:, 0], g["gX_detach"], rtol=1e-14)
    np.testing.assert_allclose(gvi, g["grad_v_init_detach"], rtol=1e-14)


# ----------------------------------------------------------------------------- P8

def _delta_expit(alpha, u):
    e = special.expit(alpha * u)
    return alpha * e * (1 - e)


@pytest.mark.parametrize("soft", [False, True])
def test_p8_backward_linear_regime_is_reversed_iir(soft):
    """With dV/dH == 1 the backward is the linear IIR gH[t] = gS[t] delta_t + k gH[t+1]
    (+ the carry at t = T-1), i.e. a time-reversed scipy lfilter([1], [1, -k]).
    Hard reset: no spikes and detach_reset=1.  Soft reset: detach_reset=1, spikes allowed."""
    rng = np.random.default_rng(11)
    tau, v_th = 2.0, 1.0
    p = OracleParams(tau=tau, v_th=v_th, decay_input=True, detach_reset=True, soft_reset=soft)
    k, s = 1 - 1 / tau, 1 / tau
    T, N = 20, 5
    X = rng.uniform(-0.5, 0.9 if not soft else 3.0, size=(T, N))
    r = forward(p, X)
    if not soft:
        assert r["S"].sum() == 0
    else:
        assert r["S"].sum() > 0
    gS = rng.normal(size=(T, N))
    gvf = rng.normal(size=N)
    gX, gvi = backward(p, gS, r["H"], grad_v_final=gvf)
    drive = gS * _delta_expit(p.alpha, r["H"] - v_th)
    drive[-1] += gvf
    gH = signal.lfilter([1.0], [1.0, -k], drive[::-1], axis=0)[::-1]
    np.testing.assert_allclose(gX, s * gH, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(gvi, k * gH[0], rtol=1e-12, atol=1e-15)


# ----------------------------------------------------------------------------- P9

def _smoothed_loss(p, X, v0, W, wv):
    r = forward(p, X, v_init=v0)
    return float((W * r["S"]).sum() + (wv * r["v_final"]).sum())


@pytest.mark.parametrize("surr", ["sigmoid", "atan"])
@pytest.mark.parametrize("soft", [False, True])
@pytest.mark.parametrize("decay_input", [False, True])
def test_p9_backward_is_exact_derivative_of_smoothed_model(surr, soft, decay_input):
    """Smoothed mode (Heaviside -> surrogate primitive everywhere) makes the backward the
    exact derivative of L = sum W*S + w_v . V_final; check by central differences."""
    rng = np.random.default_rng(3 + 2 * soft + decay_input)
    p = OracleParams(tau=1.7, v_th=1.0, v_reset=0.2, soft_reset=soft, decay_input=decay_input,
                     surrogate=surr, alpha=2.5, smoothed=True)
    T, N = 6, 3
    X = rng.uniform(0.5, 2.5, size=(T, N)) * (0.6 if not decay_input else 1.0)
    v0 = np.full(N, 0.1)
    W = rng.normal(size=(T, N))
    wv = rng.normal(size=N)
    r = forward(p, X, v_init=v0)
    gX, gvi = backward(p, W, r["H"], grad_v_final=wv)
    h = 1e-6
    fd = np.zeros((T, N))
    for t in range(T):
        for n in range(N):
            Xp = X.copy(); Xp[t, n] += h
            Xm = X.copy(); Xm[t, n] -= h
            fd[t, n] = (_smoothed_loss(p, Xp, v0, W, wv) - _smoothed_loss(p, Xm, v0, W, wv)) / (2 * h)
    np.testing.assert_allclose(gX, fd, rtol=2e-6, atol=2e-8)
    fdv = np.zeros(N)
    for n in range(N):
        vp = v0.copy(); vp[n] += h
        vm = v0.copy(); vm[n] -= h
        fdv[n] = (_smoothed_loss(p, X, vp, W, wv) - _smoothed_loss(p, X, vm, W, wv)) / (2 * h)
    np.testing.assert_allclose(gvi, fdv, rtol=2e-6, atol=2e-8)


# ----------------------------------------------------------------------------- paper literal

def test_paper_mode_equals_literal_eq1_eq2():
    """At V_reset = 0, decay_input = 0, hard reset the oracle is the paper's Eq. 1-2
     written literally: v^t = k v^{t-1}(1 - y^{t-1}) + V_rest y^{t-1} + x^t."""
    rng = np.random.default_rng(5)
    T, N = 64, 300
    x = rng.normal(size=(T, N))
    k = 1 - 1 / PAPER.tau
    v = np.zeros(N); y = np.zeros(N)
    V_lit = np.empty((T, N)); Y_lit = np.empty((T, N))
    for t in range(T):
        v = k * v * (1 - y) + 0.0 * y + x[t]
        y = (v - PAPER.v_th >= 0).astype(np.float64)
        V_lit[t] = v; Y_lit[t] = y
    r = forward(PAPER, x)
    np.testing.assert_array_equal(r["S"], Y_lit)
    np.testing.assert_allclose(r["H"], V_lit, rtol=1e-12, atol=1e-14)


def test_paper_mode_equals_literal_eq3():
    """Paper mode backward is Eq. 3 written literally, with
    grad v^{t+1} = grad x^{t+1} (dv/dx = 1 in Eq. 1) and delta(u) from scipy's expit."""
    rng = np.random.default_rng(6)
    T, N = 40, 200
    x = rng.normal(size=(T, N))
    gy = rng.normal(size=(T, N))
    r = forward(PAPER, x)
    v, y = r["H"], r["S"]
    k = 1 - 1 / PAPER.tau
    d = _delta_expit(PAPER.alpha, v - PAPER.v_th)
    gx = np.empty((T, N)); nxt = np.zeros(N)
    for t in range(T - 1, -1, -1):
        gx[t] = k * nxt * (1 - y[t] - v[t] * d[t]) + gy[t] * d[t]
        nxt = gx[t]
    gX, _ = backward(PAPER, gy, v)
    np.testing.assert_allclose(gX, gx, rtol=1e-11, atol=1e-13)


# ----------------------------------------------------------------------------- P10-P12

def test_p10_backward_linearity():
    rng = np.random.default_rng(8)
    T, N = 30, 40
    r = forward(CFG0, rng.normal(1.0, 1.0, size=(T, N)))
    gS = rng.normal(size=(T, N)); gvf = rng.normal(size=N)
    gX, gvi = backward(CFG0, gS, r["H"], gvf)
    gX2, gvi2 = backward(CFG0, 4.0 * gS, r["H"], 4.0 * gvf)   # power of 2: exact scaling
    np.testing.assert_array_equal(gX2, 4.0 * gX)
    np.testing.assert_array_equal(gvi2, 4.0 * gvi)


def test_p11_neuron_independence():
    rng = np.random.default_rng(9)
    T, N = 25, 64
    X = rng.normal(1.0, 1.0, size=(T, N)); gS = rng.normal(size=(T, N))
    r = forward(CFG0, X)
    gX, gvi = backward(CFG0, gS, r["H"])
    perm = rng.permutation(N)
    rp = forward(CFG0, X[:, perm])
    np.testing.assert_array_equal(rp["H"], r["H"][:, perm])
    gXp, gvip = backward(CFG0, gS[:, perm], rp["H"])
    np.testing.assert_array_equal(gXp, gX[:, perm])
    sub = np.array([3, 17, 40])
    rs = forward(CFG0, X[:, sub])
    np.testing.assert_array_equal(rs["S"], r["S"][:, sub])


@pytest.mark.parametrize("cuts", [[1], [5, 6], [3, 11, 19], [23]])
def test_p12_segmentation_soundness(cuts):
    """Chained segments (v_final -> v_init forward, grad_v_init -> grad_v_final backward)
    equal the whole axis."""
    rng = np.random.default_rng(10)
    T, N = 24, 33
    p = OracleParams(tau=1.6, v_th=0.8, v_reset=0.1, soft_reset=False, decay_input=True)
    X = rng.normal(0.8, 1.0, size=(T, N)); gS = rng.normal(size=(T, N))
    whole = forward(p, X)
    gX_w, gvi_w = backward(p, gS, whole["H"])
    bounds = [0] + cuts + [T]
    v = None; Hs = []; Ss = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        seg = forward(p, X[a:b], v_init=v)
        v = seg["v_final"]; Hs.append(seg["H"]); Ss.append(seg["S"])
    np.testing.assert_array_equal(np.concatenate(Hs), whole["H"])
    np.testing.assert_array_equal(np.concatenate(Ss), whole["S"])
    np.testing.assert_array_equal(v, whole["v_final"])
    g = None; gXs = []
    for a, b, H in reversed(list(zip(bounds[:-1], bounds[1:], Hs))):
        gx, g = backward(p, gS[a:b], H, grad_v_final=g)
        gXs.insert(0, gx)
    np.testing.assert_array_equal(np.concatenate(gXs), gX_w)
    np.testing.assert_array_equal(g, gvi_w)


# ----------------------------------------------------------------------------- edges

def test_nan_input_propagates():
    """a NaN current gives S = 0 and NaN H / V from then on."""
    x = np.array([[0.5], [np.nan], [0.5]])
    r = forward(PAPER, x)
    assert r["S"][1, 0] == 0 and np.isnan(r["H"][1, 0]) and np.isnan(r["H"][2, 0])


def test_t1_n1_and_empty_carry_defaults():
    r = forward(CFG0, col(2.0, 1))
    assert r["H"][0, 0] == 1.0 and r["S"][0, 0] == 1.0 and r["v_final"][0] == 0.0
    gX, gvi = backward(CFG0, np.ones((1, 1)), r["H"])
    assert gX[0, 0] == pytest.approx(0.5)   # s * delta(0) = 0.5 * 1
    assert gvi[0] == pytest.approx(0.5 * 1.0)


# ----------------------------------------------------------------------------- affine prologue (f4)

from oracle import affine_grads, affine_input  # noqa: E402


def test_affine_identity_and_channel_map():
    rng = np.random.default_rng(21)
    T, B, C, HW = 3, 2, 3, 4
    x = rng.normal(size=(T, B * C * HW))
    np.testing.assert_array_equal(affine_input(x, np.ones(C), np.zeros(C), C, HW), x)
    scale = np.array([2.0, -1.0, 0.5]); shift = np.array([0.25, 0.0, -1.0])
    xp = affine_input(x, scale, shift, C, HW)
    xr = x.reshape(T, B, C, HW)       # independent reshape-based definition of c(n)
    np.testing.assert_allclose(xp, (xr * scale[None, None, :, None] + shift[None, None, :, None]).reshape(T, -1))


@pytest.mark.parametrize("decay_input", [False, True])
def test_affine_gradients_finite_differences(decay_input):
    """Smoothed model: L(scale, shift, X) = sum W*S + w_v . V_final with the LIF input
    X' = scale[c] X + shift[c]; oracle backward + affine_grads vs central differences."""
    rng = np.random.default_rng(22)
    T, B, C, HW = 5, 2, 2, 3
    N = B * C * HW
    p = OracleParams(tau=1.6, v_th=0.7, v_reset=0.1, decay_input=decay_input, alpha=2.5, smoothed=True)
    X = rng.uniform(-0.5, 1.5, size=(T, N))
    scale = np.array([1.3, 0.8]); shift = np.array([0.2, -0.1])
    W = rng.normal(size=(T, N)); wv = rng.normal(size=N)

    def loss(sc, sh, xx):
        r = forward(p, affine_input(xx, sc, sh, C, HW))
        return float((W * r["S"]).sum() + (wv * r["v_final"]).sum())

    r = forward(p, affine_input(X, scale, shift, C, HW))
    gxp, _ = backward(p, W, r["H"], grad_v_final=wv)
    gx, gs, gb = affine_grads(X, gxp, scale, C, HW)
    h = 1e-6
    for c in range(C):
        e = np.zeros(C); e[c] = h
        assert gs[c] == pytest.approx((loss(scale + e, shift, X) - loss(scale - e, shift, X)) / (2 * h), rel=2e-6, abs=1e-8)
        assert gb[c] == pytest.approx((loss(scale, shift + e, X) - loss(scale, shift - e, X)) / (2 * h), rel=2e-6, abs=1e-8)
    for (t, n) in [(0, 0), (2, 5), (4, 11)]:
        Xp = X.copy(); Xp[t, n] += h
        Xm = X.copy(); Xm[t, n] -= h
        assert gx[t, n] == pytest.approx((loss(scale, shift, Xp) - loss(scale, shift, Xm)) / (2 * h), rel=2e-6, abs=1e-8)


def test_affine_residual_input_definition():
    """X' = scale[c] X + shift[c] + R: reduces to the plain affine at R = 0, to R itself at
    scale = 0, shift = 0, and equals an independent reshape-based evaluation."""
    rng = np.random.default_rng(23)
    T, B, C, HW = 3, 2, 3, 4
    x = rng.normal(size=(T, B * C * HW))
    R = rng.normal(size=x.shape)
    scale = np.array([2.0, -1.0, 0.5]); shift = np.array([0.25, 0.0, -1.0])
    np.testing.assert_array_equal(affine_input(x, scale, shift, C, HW, residual=np.zeros_like(x)),
                                  affine_input(x, scale, shift, C, HW))
    np.testing.assert_array_equal(affine_input(x, np.zeros(C), np.zeros(C), C, HW, residual=R), R)
    xr = x.reshape(T, B, C, HW)
    ref = (xr * scale[None, None, :, None] + shift[None, None, :, None]).reshape(T, -1) + R
    np.testing.assert_allclose(affine_input(x, scale, shift, C, HW, residual=R), ref, rtol=0, atol=1e-15)


@pytest.mark.parametrize("soft", [False, True])
def test_affine_residual_gradient_finite_differences(soft):
    """dL/dR = dL/dX' (the oracle backward's gX at the input X' = scale X + shift + R), and the
    affine gradients are unchanged by R: central differences of the smoothed model in R,
    scale and X."""
    rng = np.random.default_rng(24)
    T, B, C, HW = 4, 2, 2, 3
    N = B * C * HW
    p = OracleParams(tau=1.4, v_th=0.6, v_reset=0.0, soft_reset=soft, alpha=3.0, smoothed=True)
    X = rng.uniform(-0.5, 1.0, size=(T, N))
    R = rng.uniform(-0.5, 0.8, size=(T, N))
    scale = np.array([1.1, 0.7]); shift = np.array([0.1, -0.2])
    W = rng.normal(size=(T, N)); wv = rng.normal(size=N)

    def loss(sc, xx, rr):
        r = forward(p, affine_input(xx, sc, shift, C, HW, residual=rr))
        return float((W * r["S"]).sum() + (wv * r["v_final"]).sum())

    r = forward(p, affine_input(X, scale, shift, C, HW, residual=R))
    gxp, _ = backward(p, W, r["H"], grad_v_final=wv)
    gx, gs, _ = affine_grads(X, gxp, scale, C, HW)
    h = 1e-6
    for (t, n) in [(0, 0), (1, 7), (3, 11)]:
        Rp = R.copy(); Rp[t, n] += h
        Rm = R.copy(); Rm[t, n] -= h
        assert gxp[t, n] == pytest.approx((loss(scale, X, Rp) - loss(scale, X, Rm)) / (2 * h), rel=2e-6, abs=1e-8)
        Xp = X.copy(); Xp[t, n] += h
        Xm = X.copy(); Xm[t, n] -= h
        assert gx[t, n] == pytest.approx((loss(scale, Xp, R) - loss(scale, Xm, R)) / (2 * h), rel=2e-6, abs=1e-8)
    e = np.array([h, 0.0])
    assert gs[0] == pytest.approx((loss(scale + e, X, R) - loss(scale - e, X, R)) / (2 * h), rel=2e-6, abs=1e-8)
