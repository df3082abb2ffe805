"""Multi-process host logic of the N>1 paths on CPU (gloo, world_size 2-3): the SPEC
partition rule, Eq. 5, neuron shards, the time-segment pipeline protocol (driven by the
oracle as the per-segment compute) and the max-over-ranks timing reduction."""
import math
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import importlib.util
import sys

from conftest import ROOT

# paper_2408_00280_b200/dist.py is pure host logic; load it without importing the package
# (which loads the CUDA library) so these tests run on a CPU-only box.
_spec = importlib.util.spec_from_file_location("snn_dist", os.path.join(ROOT, "paper_2408_00280_b200", "dist.py"))
D = importlib.util.module_from_spec(_spec)
import sys  # noqa: E402
sys.modules["snn_dist"] = D
_spec.loader.exec_module(D)


# ----------------------------------------------------------------------------- partitions

def test_partition_time_spec_examples():
    lens = lambda segs: [b - a for a, b in segs]
    assert lens(D.partition_time(32, 4)) == [8, 8, 8, 8]
    assert lens(D.partition_time(10, 3)) == [4, 3, 3]
    assert lens(D.partition_time(5, 5)) == [1, 1, 1, 1, 1]
    for T in range(1, 40):
        for k in range(1, T + 1):
            segs = D.partition_time(T, k)
            assert segs[0][0] == 0 and segs[-1][1] == T
            assert all(a < b for a, b in segs)
            assert all(s[1] == n[0] for s, n in zip(segs, segs[1:]))
            assert max(lens(segs)) - min(lens(segs)) <= 1
    with pytest.raises(ValueError):
        D.partition_time(3, 4)
    with pytest.raises(ValueError):
        D.partition_time(3, 0)


def test_shard_range_and_chunks_cover_disjointly():
    for N in [1, 7, 512, 1000, 4096, 12345]:
        for w in [1, 2, 3, 8]:
            rs = [D.shard_range(N, w, r, align=4) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(lo % 4 == 0 or lo == N for lo, _ in rs)
    ch = D.neuron_chunks(4 << 20, 32)
    assert len(ch) == 32 and all((b - a) == (4 << 20) // 32 for a, b in ch)


# ----------------------------------------------------------------------------- Eq. 5

def test_eq5_closed_forms():
    assert D.speedup_mu(16.0, 1.0, 1) == 1.0                        # mu(k=1) = 1
    assert D.speedup_mu(16.0, 1.0, 4) == pytest.approx(16 / 7)
    assert D.optimal_k(16.0, 1.0) == 4.0
    assert D.optimal_k(3.0, 3.0) == 1.0
    assert D.speedup_mu(64.0, 1.0, 8) == pytest.approx(4.2667, abs=1e-4)


@pytest.mark.parametrize("ratio", [2.0, 4.0, 16.0, 64.0, 650.0])
def test_eq5_optimum_and_unimodality(ratio):
    kopt = D.optimal_k(ratio, 1.0)
    ks = range(1, int(10 * kopt) + 2)
    mus = [D.speedup_mu(ratio, 1.0, k) for k in ks]
    best = max(D.speedup_mu(ratio, 1.0, math.floor(kopt)), D.speedup_mu(ratio, 1.0, math.ceil(kopt)))
    assert best >= max(mus) - 1e-12
    peak = int(np.argmax(mus))
    assert all(mus[i] <= mus[i + 1] + 1e-12 for i in range(peak))
    assert all(mus[i] >= mus[i + 1] - 1e-12 for i in range(peak, len(mus) - 1))


def test_model_curve_rows_and_monotone_peaks():
    rows = D.model_curve([4, 16, 64], 10)
    assert len(rows) == 30 and all(mu == 1.0 for r, k, mu in rows if k == 1)
    peaks = [max(mu for r, k, mu in rows if r == ratio) for ratio in (4, 16, 64)]
    assert peaks == sorted(peaks)


def test_pipeline_efficiency():
    assert D.pipeline_efficiency(32, 8) == pytest.approx(32 / 39)
    assert D.pipeline_efficiency(1, 1) == 1.0


# ----------------------------------------------------------------------------- multi-process

def _rendezvous_file():
    import tempfile
    fd, path = tempfile.mkstemp(prefix="snn_pg_")
    os.close(fd)
    os.remove(path)   # the FileStore creates it; a fresh name per test
    return path


def _oracle_fns(op):
    import oracle

    def fwd_fn(x_chunk, v_in):
        r = oracle.forward(op, x_chunk.double().numpy(), v_init=None if v_in is None else v_in.double().numpy())
        return r["H"], torch.from_numpy(r["S"]), torch.from_numpy(r["v_final"]).float()

    def bwd_fn(g_chunk, H, g_in):
        gX, gvi = oracle.backward(op, g_chunk.double().numpy(), H,
                                  grad_v_final=None if g_in is None else g_in.double().numpy())
        return torch.from_numpy(gX), torch.from_numpy(gvi).float()

    return fwd_fn, bwd_fn


def _tsplit_worker(rank, world, port, T, N, n_chunks, out):
    # file-based rendezvous: no TCP port to race for between consecutive tests
    dist.init_process_group("gloo", init_method=f"file://{port}", rank=rank, world_size=world)
    import oracle
    import snn_synth
    # v carries are exchanged as fp32 (the product's boundary payload); the
    # oracle inputs are fp32-exact values so the chained fp64 oracle sees the same numbers
    # as a whole-axis run except for the fp32 rounding of the carried V / dV.
    op = oracle.OracleParams(tau=float(np.float32(1.6)), v_th=float(np.float32(0.8)), v_reset=0.0,
                             decay_input=True)
    a, b = D.partition_time(T, world)[rank]
    X = snn_synth.normal_tensor(7, b - a, N, t_offset=a, n_global=N, mean=0.8)
    G = snn_synth.normal_tensor(8, b - a, N, t_offset=a, n_global=N)
    ts = D.TimeSplitLIF(rank, world, D.HostTransport(), n_chunks=n_chunks, align=4)
    fwd_fn, bwd_fn = _oracle_fns(op)
    spikes, state, v_final = ts.forward(X, fwd_fn)
    gxs, gvi = ts.backward(G, state, bwd_fn)
    # gather to rank 0 for the check (host logic only)
    S = spikes.float()
    gX = gxs.float()
    objs = [None] * world
    dist.all_gather_object(objs, (a, b, S.numpy(), gX.numpy(), ts.messages_sent,
                                  None if v_final is None else v_final.numpy(),
                                  None if gvi is None else gvi.numpy()))
    # max-over-ranks reduction used by bench.py for the timed region
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out.put((objs, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_chunks", [(2, 1), (2, 4), (3, 3)])
def test_time_split_over_gloo_matches_whole_axis(world, n_chunks):
    import oracle
    import snn_synth
    T, N = 23, 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _rendezvous_file()
    procs = [ctx.Process(target=_tsplit_worker, args=(r, world, port, T, N, n_chunks, q))
             for r in range(world)]
    for p in procs:
        p.start()
    objs, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == float(world)
    # whole-axis oracle with the same fp32 boundary rounding chained segment by segment
    op = oracle.OracleParams(tau=float(np.float32(1.6)), v_th=float(np.float32(0.8)), v_reset=0.0,
                             decay_input=True)
    X = snn_synth.normal_tensor(7, T, N, mean=0.8).double().numpy()
    G = snn_synth.normal_tensor(8, T, N).double().numpy()
    objs = sorted(objs, key=lambda o: o[0])
    v = None; Hs = []
    for (a, b, S, gX, msgs, vf, gvi) in objs:
        r = oracle.forward(op, X[a:b], v_init=v)
        np.testing.assert_array_equal(S, r["S"])
        v = r["v_final"].astype(np.float32).astype(np.float64)
        Hs.append(r["H"])
    g = None
    for (a, b, S, gX, msgs, vf, gvi), H in reversed(list(zip(objs, Hs))):
        ref, g = oracle.backward(op, G[a:b], H, grad_v_final=g)
        np.testing.assert_allclose(gX, ref, rtol=1e-6, atol=1e-7)
        g = g.astype(np.float32).astype(np.float64)
    # protocol liveness: exactly one message per boundary per chunk per direction
    n_eff = len(D.neuron_chunks(N, n_chunks, 4))
    sent = [o[4] for o in objs]
    assert sent[0] == n_eff and sent[-1] == n_eff
    assert sum(sent) == 2 * (world - 1) * n_eff
    assert objs[-1][5] is not None and objs[0][6] is not None


# ----------------------------------------------------------------------------- f3 pipeline

def _load_pipeline():
    """pipeline.py imports `.dist`; provide it as a package-less module pair."""
    import types
    pkg = types.ModuleType("snn_pkg_cpu")
    pkg.__path__ = []
    sys.modules["snn_pkg_cpu"] = pkg
    sys.modules["snn_pkg_cpu.dist"] = D
    spec = importlib.util.spec_from_file_location("snn_pkg_cpu.pipeline",
                                                  os.path.join(ROOT, "paper_2408_00280_b200", "pipeline.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["snn_pkg_cpu.pipeline"] = mod
    spec.loader.exec_module(mod)
    return mod


def _build_model(P, rank, world, transport, op, seed=0):
    torch.manual_seed(seed)
    fwd_fn, bwd_fn = _oracle_fns(op)
    lin1 = torch.nn.Linear(24, 40)
    lin2 = torch.nn.Linear(40, 5)
    return torch.nn.Sequential(P.TimeFolded(lin1),
                               P.TimeSplitLIFLayer(rank, world, transport, fwd_fn, bwd_fn, n_chunks=3, align=4),
                               P.TimeFolded(lin2))


def _pipeline_worker(rank, world, path, T, out):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    import oracle
    import snn_synth
    P = _load_pipeline()
    op = oracle.OracleParams(tau=float(np.float32(1.25)), v_th=float(np.float32(0.3)), v_reset=0.0)
    a, b = D.partition_time(T, world)[rank]
    x = snn_synth.normal_tensor(91, b - a, 8 * 24, t_offset=a, n_global=8 * 24).reshape(b - a, 8, 24)
    target = torch.arange(8) % 5
    model = _build_model(P, rank, world, D.HostTransport(), op)
    tr = P.TimeSplitTrainer(model, T)
    loss = tr.step(x, torch.nn.functional.cross_entropy, target)
    grads = [p.grad.detach().numpy().copy() for p in model.parameters()]
    if rank == 0:
        out.put((float(loss), grads))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_layer_pipelined_time_split_training_step_equals_whole_axis(world):
    """SURVEY f3 / Fig. 1(b): Linear -> time-split LIF -> Linear, rate-coded cross-entropy.
    k ranks each own a time segment of every layer; loss and (all-reduced) weight gradients
    equal one whole-axis step (oracle as the LIF compute; gloo on CPU)."""
    import oracle
    import snn_synth
    T = 13
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    path = _rendezvous_file()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, world, path, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    loss_k, grads_k = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P = _load_pipeline()
    op = oracle.OracleParams(tau=float(np.float32(1.25)), v_th=float(np.float32(0.3)), v_reset=0.0)
    x = snn_synth.normal_tensor(91, T, 8 * 24).reshape(T, 8, 24)
    model = _build_model(P, 0, 1, None, op)
    loss_1 = P.TimeSplitTrainer(model, T).step(x, torch.nn.functional.cross_entropy, torch.arange(8) % 5)
    assert loss_k == pytest.approx(float(loss_1), rel=1e-6)
    for gk, p in zip(grads_k, model.parameters()):
        np.testing.assert_allclose(gk, p.grad.numpy(), rtol=1e-5, atol=1e-6)
