"""Launch scheduling never changes results (r2b): the work distribution of the TMA kernels --
steal requests in flight (SNN_LIF_CLC_DEPTH), the L2 prefetch before griddepcontrol.wait
(SNN_LIF_PREFETCH) -- only changes which CTA runs a tile and when, so spikes, dL/dX and the
carries must be bitwise identical under every setting, and equal to the oracle on sampled
columns.  The knobs are read once per process, so each setting runs in a subprocess."""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import hashlib, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2408_00280_b200 as snn, snn_synth
p = snn.LIFParams.paper()
h = hashlib.sha256()
for dt, T, N in ((torch.float32, 24, 600_000), (torch.bfloat16, 16, 1_200_000), (torch.float32, 200, 300_032)):
    X = snn_synth.normal_tensor(1234, T, N, device="cuda", dtype=dt)
    G = snn_synth.normal_tensor(4321, T, N, device="cuda", dtype=dt)
    for fmt in ("u8", "bits"):
        f = snn.lif_forward(X, p, spike_fmt=fmt)
        gx, gv = snn.lif_backward(G, f)
        torch.cuda.synchronize()
        for t in (f.spikes, f.v_final, gx, gv):
            h.update(t.contiguous().view(torch.uint8).cpu().numpy().tobytes())
print(h.hexdigest())
"""

SETTINGS = [{}, {"SNN_LIF_CLC_DEPTH": "4"}, {"SNN_LIF_PREFETCH": "0"}, {"SNN_LIF_PREFETCH": "64"}]


def _digest(env):
    e = dict(os.environ)
    e.update(env)
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=e, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


def test_scheduling_knobs_do_not_change_results():
    digests = [_digest(s) for s in SETTINGS]
    assert all(d == digests[0] for d in digests), dict(zip(map(str, SETTINGS), digests))


def test_many_tile_grid_matches_oracle_on_sampled_columns():
    """The default scheduling on a grid several times the resident CTAs (work stealing active,
    short tiles prefetched): sampled columns against the oracle."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import paper_2408_00280_b200 as snn
    import snn_synth
    from parity import oracle_check
    p = snn.LIFParams.paper()
    T, N = 24, 600_000
    X = snn_synth.normal_tensor(1234, T, N, device="cuda")
    G = snn_synth.normal_tensor(4321, T, N, device="cuda")
    f = snn.lif_forward(X, p)
    gx, gv = snn.lif_backward(G, f)
    torch.cuda.synchronize()
    cols = np.sort(np.random.default_rng(7).choice(N, 2048, replace=False))
    c = torch.from_numpy(cols)
    rep = oracle_check(p, X.cpu()[:, c], G.cpu()[:, c], f.spikes.cpu()[:, c], gx.cpu()[:, c],
                       vf_gpu=f.v_final.cpu()[c], gvi_gpu=gv.cpu()[c])
    assert rep.ok, str(rep)


@pytest.mark.parametrize("tiles_fwd", [295, 296, 297, 593])
def test_grid_sizes_around_the_resident_count_equal_generic(monkeypatch, tiles_fwd):
    """Grids just below / at / just above the resident CTA count (148 SMs x 2 forward CTAs of
    1024 neurons; the backward's 512-neuron tiles give twice the count at 1 CTA/SM): no steal,
    exactly one steal, and a second wave -- the TMA kernels equal the generic kernels bitwise."""
    import paper_2408_00280_b200 as snn
    import snn_synth
    p = snn.LIFParams.paper()
    T, N = 20, tiles_fwd * 1024
    X = snn_synth.normal_tensor(1234, T, N, device="cuda")
    G = snn_synth.normal_tensor(4321, T, N, device="cuda")
    outs = []
    for no_tma in ("0", "1"):
        monkeypatch.setenv("SNN_LIF_NO_TMA", no_tma)
        f = snn.lif_forward(X, p)
        gx, gv = snn.lif_backward(G, f)
        torch.cuda.synchronize()
        outs.append((f.spikes, f.v_final, gx, gv))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
