"""snn_lif_plan_*: a recorded layer call replays the same kernels -- bitwise equal to the
direct calls -- on the TMA and generic paths, with in-place input updates between replays."""
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_00280_b200 as snn  # noqa: E402
import snn_synth  # noqa: E402

P = snn.LIFParams.paper()


@pytest.mark.parametrize("T,N,dtype,save_mode,spike_fmt", [
    (64, 4096, torch.float32, "recompute", "u8"), (33, 3001, torch.float32, "h", "bits"),
    (16, 8192, torch.bfloat16, "recompute", "io"), (7, 1000, torch.bfloat16, "h", "u8")])
def test_plan_replay_equals_direct_calls_bitwise(T, N, dtype, save_mode, spike_fmt):
    X = snn_synth.normal_tensor(51, T, N, dtype=dtype, device="cuda")
    G = snn_synth.normal_tensor(52, T, N, dtype=dtype, device="cuda")
    v0 = snn_synth.normal_tensor(53, 1, N, std=0.2, device="cuda")[0]
    gvf = snn_synth.normal_tensor(54, 1, N, device="cuda")[0]
    x_buf, g_buf = torch.zeros_like(X), torch.zeros_like(G)
    plan = snn.LIFPlan(x_buf, P, spike_fmt=spike_fmt, save_mode=save_mode, v_init=v0, grad_spikes=g_buf,
                       grad_v_final=gvf, with_v_final=True, with_grad_v_init=True)
    for it in range(3):                       # new contents, same buffers, every replay
        Xi, Gi = X * (1.0 + 0.1 * it), G - 0.05 * it
        x_buf.copy_(Xi); g_buf.copy_(Gi)
        s = plan.forward().clone()
        gx = plan.backward().clone()
        f = snn.lif_forward(Xi, P, v_init=v0, spike_fmt=spike_fmt, save_mode=save_mode)
        gx_ref, gvi_ref = snn.lif_backward(Gi, f, grad_v_final=gvf)
        torch.cuda.synchronize()
        assert torch.equal(s, f.spikes) and torch.equal(plan.v_final, f.v_final)
        assert torch.equal(gx, gx_ref) and torch.equal(plan.grad_v_init, gvi_ref)


def test_forward_only_plan_and_errors():
    X = torch.randn(8, 512, device="cuda")
    plan = snn.LIFPlan(X, P, save_mode="none")
    s = plan.forward()
    f = snn.lif_forward(X, P, save_mode="none")
    torch.cuda.synchronize()
    assert torch.equal(s, f.spikes)
    with pytest.raises(RuntimeError, match="INVALID_VALUE"):
        plan.backward()
    with pytest.raises(RuntimeError, match="INVALID_VALUE"):   # validated at creation, like the direct call
        snn.LIFPlan(X, snn.LIFParams(tau=1.0, v_th=0.0, v_reset=0.0))


def test_plan_inside_cuda_graph():
    """A plan's replay is capturable: forward + backward captured once, replayed with new data."""
    T, N = 32, 4096
    x_buf = torch.zeros(T, N, device="cuda"); g_buf = torch.zeros(T, N, device="cuda")
    plan = snn.LIFPlan(x_buf, P, grad_spikes=g_buf)
    plan.forward(); plan.backward(); torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        plan.forward(); plan.backward()
    X = snn_synth.normal_tensor(61, T, N, device="cuda"); G = snn_synth.normal_tensor(62, T, N, device="cuda")
    x_buf.copy_(X); g_buf.copy_(G)
    graph.replay()
    f = snn.lif_forward(X, P); gx, _ = snn.lif_backward(G, f)
    torch.cuda.synchronize()
    assert torch.equal(plan.spikes, f.spikes) and torch.equal(plan.grad_x, gx)


@pytest.mark.parametrize("residual", [False, True])
def test_affine_plan_equals_direct_calls_bitwise(residual):
    T, B, C, HW = 24, 4, 8, 64
    N = B * C * HW
    X = snn_synth.normal_tensor(71, T, N, device="cuda")
    G = snn_synth.normal_tensor(72, T, N, device="cuda")
    R = snn_synth.normal_tensor(73, T, N, std=0.5, device="cuda") if residual else None
    af = snn.AffineSpec(torch.linspace(0.5, 1.5, C, device="cuda"), torch.linspace(-0.2, 0.2, C, device="cuda"),
                        C, HW)
    x_buf, g_buf = X.clone(), G.clone()
    r_buf = None if R is None else R.clone()
    plan = snn.LIFPlan(x_buf, P, grad_spikes=g_buf, affine=af, residual=r_buf, with_v_final=True)
    s = plan.forward().clone(); gx = plan.backward().clone()
    f = snn.lif_forward_affine(X, P, af, residual=R)
    out = snn.lif_backward_affine(G, f)
    torch.cuda.synchronize()
    assert torch.equal(s, f.spikes) and torch.equal(plan.v_final, f.v_final)
    assert torch.equal(gx, out[0]) and torch.equal(plan.grad_scale, out[2]) and torch.equal(plan.grad_shift, out[3])
    if residual:
        assert torch.equal(plan.grad_residual, out[4])
    inf = snn.LIFPlan(x_buf, P, save_mode="none", affine=af, residual=r_buf)   # BN-folded inference
    s2 = inf.forward()
    torch.cuda.synchronize()
    assert torch.equal(s2, f.spikes)


from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402


@settings(max_examples=25, deadline=None, derandomize=True, suppress_health_check=list(HealthCheck))
@given(T=st.integers(1, 40), N=st.integers(1, 3000), dtype=st.sampled_from([torch.float32, torch.bfloat16]),
       mode=st.integers(0, 7), decay_input=st.booleans(), v_reset=st.sampled_from([0.0, 0.1]),
       save_mode=st.sampled_from(["recompute", "h"]), spike_fmt=st.sampled_from(["u8", "bits", "io"]))
def test_randomized_plan_equals_direct(T, N, dtype, mode, decay_input, v_reset, save_mode, spike_fmt):
    """Random shapes (TMA and generic paths), every reset/surrogate/detach mode, paper-mode and
    general constants: a plan's replay is bitwise the direct calls."""
    p = snn.LIFParams(tau=1.5, v_th=0.6, v_reset=v_reset, surrogate=("atan" if mode & 1 else "sigmoid"),
                      reset=("soft" if mode & 2 else "hard"), detach_reset=bool(mode & 4),
                      decay_input=decay_input, alpha=(2.0 if mode & 1 else 4.0))
    X = snn_synth.normal_tensor(T * 31 + N, T, N, mean=0.5, dtype=dtype, device="cuda")
    G = snn_synth.normal_tensor(T * 37 + N, T, N, dtype=dtype, device="cuda")
    plan = snn.LIFPlan(X, p, spike_fmt=spike_fmt, save_mode=save_mode, grad_spikes=G, with_v_final=True,
                       with_grad_v_init=True)
    s = plan.forward().clone(); gx = plan.backward().clone()
    f = snn.lif_forward(X, p, spike_fmt=spike_fmt, save_mode=save_mode)
    gx_ref, gvi_ref = snn.lif_backward(G, f)
    torch.cuda.synchronize()
    assert torch.equal(s, f.spikes) and torch.equal(plan.v_final, f.v_final)
    assert torch.equal(gx, gx_ref) and torch.equal(plan.grad_v_init, gvi_ref)
