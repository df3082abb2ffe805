"""Time-segment split with the CUDA kernels: k processes share cuda:0 and exchange the
boundary V / dV through HostTransport (gloo); the result must be BITWISE equal to one
whole-axis run (segmented execution carries exactly the register state)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _rendezvous_file():
    import tempfile
    fd, path = tempfile.mkstemp(prefix="snn_pg_")
    os.close(fd)
    os.remove(path)   # the FileStore creates it; a fresh name per test
    return path


def _worker(rank, world, port, T, N, n_chunks, dtype, out, backend="gloo"):
    # file-based rendezvous: no TCP port to race for between consecutive tests
    if backend == "nccl":   # two ranks on one GPU: distinct NCCL host ids -> socket transport
        os.environ.update(NCCL_HOSTID=f"snn-dist-host-{rank}", NCCL_P2P_DISABLE="1", NCCL_SHM_DISABLE="1",
                          NCCL_IB_DISABLE="1", NCCL_NET="Socket", NCCL_SOCKET_IFNAME="lo", NCCL_NVLS_ENABLE="0")
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", init_method=f"file://{port}", rank=rank, world_size=world,
                                device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", init_method=f"file://{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2408_00280_b200 as snn
    from paper_2408_00280_b200 import dist as D
    import snn_synth
    p = snn.LIFParams.paper()
    a, b = D.partition_time(T, world)[rank]
    X = snn_synth.normal_tensor(1234, b - a, N, t_offset=a, dtype=dtype, device="cuda")
    G = snn_synth.normal_tensor(4321, b - a, N, t_offset=a, dtype=dtype, device="cuda")
    transport = D.NcclTransport() if backend == "nccl" else D.HostTransport()
    ts = D.TimeSplitLIF(rank, world, transport, n_chunks=n_chunks)
    fwd_fn, bwd_fn = D.lif_segment_fns(p)
    spikes, state, v_final = ts.forward(X, fwd_fn)
    gxs, gvi = ts.backward(G, state, bwd_fn)
    torch.cuda.synchronize()
    objs = [None] * world
    # numpy (pickled by value): a torch CPU tensor put on an mp.Queue is shared through a
    # file-descriptor socket that dies with this process, racing the parent's get().
    np_ = lambda t: None if t is None else t.cpu().view(torch.int16 if t.dtype == torch.bfloat16 else t.dtype).numpy()
    dist.all_gather_object(objs, (a, b, np_(spikes), np_(gxs),
                                  np_(v_final), np_(gvi)))
    if rank == 0:
        out.put(objs)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_chunks,dtype,backend", [(2, 4, torch.float32, "gloo"), (4, 3, torch.float32, "gloo"),
                                                          (3, 2, torch.bfloat16, "gloo"), (2, 3, torch.float32, "nccl")])
def test_time_split_bitwise_equals_whole_axis(world, n_chunks, dtype, backend):
    """backend "nccl": the NcclTransport (torch.distributed isend / irecv over NCCL) between two
    ranks on this one GPU (distinct NCCL host ids, socket transport)."""
    import paper_2408_00280_b200 as snn
    import snn_synth
    T, N = 70, 4096
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _rendezvous_file()
    ps = [ctx.Process(target=_worker, args=(r, world, port, T, N, n_chunks, dtype, q, backend), daemon=True)
          for r in range(world)]
    for p in ps:
        p.start()
    try:
        objs = sorted(q.get(timeout=300), key=lambda o: o[0])
        for p in ps:
            p.join(timeout=60)
            assert p.exitcode == 0
    finally:
        for p in ps:
            if p.is_alive():
                p.kill()
    X = snn_synth.normal_tensor(1234, T, N, dtype=dtype, device="cuda")
    G = snn_synth.normal_tensor(4321, T, N, dtype=dtype, device="cuda")
    f = snn.lif_forward(X, snn.LIFParams.paper())
    gx, gvi = snn.lif_backward(G, f)
    torch.cuda.synchronize()
    as_np = lambda t: t.cpu().view(torch.int16 if t.dtype == torch.bfloat16 else t.dtype).numpy()
    assert np.array_equal(np.concatenate([o[2] for o in objs], 0), as_np(f.spikes))
    assert np.array_equal(np.concatenate([o[3] for o in objs], 0), as_np(gx))   # bitwise (int16 view for bf16)
    assert np.array_equal(objs[-1][4], as_np(f.v_final))
    assert np.array_equal(objs[0][5], as_np(gvi))
    # ... and anchored to the oracle directly (not only to the whole-axis CUDA run): the
    # k-rank result vs the fp64 oracle on the host-regenerated inputs.
    from parity import oracle_check
    to_t = lambda a: (torch.from_numpy(a).view(torch.bfloat16).float() if dtype == torch.bfloat16
                      else torch.from_numpy(a))
    rep = oracle_check(snn.LIFParams.paper(), snn_synth.normal_tensor(1234, T, N, dtype=dtype),
                       snn_synth.normal_tensor(4321, T, N, dtype=dtype),
                       torch.from_numpy(np.concatenate([o[2] for o in objs], 0)),
                       to_t(np.concatenate([o[3] for o in objs], 0)),
                       vf_gpu=torch.from_numpy(objs[-1][4]), gvi_gpu=torch.from_numpy(objs[0][5]),
                       io_bf16=dtype == torch.bfloat16)
    assert rep.ok, str(rep)


def _pipe_worker(rank, world, path, T, out):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2408_00280_b200 as snn
    from paper_2408_00280_b200 import dist as D, pipeline as P
    import snn_synth
    torch.manual_seed(0)
    fwd_fn, bwd_fn = D.lif_segment_fns(snn.LIFParams.paper(), spike_fmt="io")
    model = torch.nn.Sequential(
        P.TimeFolded(torch.nn.Conv2d(2, 16, 3, padding=1)),
        P.TimeSplitLIFLayer(rank, world, D.HostTransport(), fwd_fn, bwd_fn, n_chunks=2),
        P.TimeFolded(torch.nn.Flatten()), P.TimeFolded(torch.nn.Linear(16 * 16 * 16, 10))).cuda()
    a, b = D.partition_time(T, world)[rank]
    x = snn_synth.normal_tensor(93, b - a, 4 * 2 * 16 * 16, t_offset=a, device="cuda").reshape(b - a, 4, 2, 16, 16)
    # the LIF layer's own input / output / gradients on this rank's segment (for the oracle check)
    seen = {}
    lif = model[1]
    lif.register_forward_hook(lambda m, i, o: seen.update(x=i[0].detach().reshape(b - a, -1).cpu().numpy(),
                                                          s=o.detach().reshape(b - a, -1).cpu().numpy()))
    lif.register_full_backward_hook(lambda m, gi, go: seen.update(gx=gi[0].detach().reshape(b - a, -1).cpu().numpy(),
                                                                  gs=go[0].detach().reshape(b - a, -1).cpu().numpy()))
    loss = P.TimeSplitTrainer(model, T).step(x, torch.nn.functional.cross_entropy,
                                            torch.arange(4, device="cuda") % 10)
    grads = [p.grad.detach().cpu().numpy() for p in model.parameters()]
    segs = [None] * world
    dist.all_gather_object(segs, (a, seen["x"], seen["s"], seen["gs"], seen["gx"]))
    if rank == 0:
        out.put((float(loss), grads, sorted(segs, key=lambda q: q[0])))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_conv_snn_time_split_training_step(world):
    """SURVEY f3 / Fig. 1(b) with the CUDA kernels: Conv -> time-split LIF -> Linear,
    k processes own time segments of every layer; loss and all-reduced weight gradients
    match one whole-axis step (conv/linear run on different batch sizes, so tolerance)."""
    import paper_2408_00280_b200 as snn
    from paper_2408_00280_b200 import dist as D, pipeline as P
    import snn_synth
    T = 20
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    path = _rendezvous_file()
    ps = [ctx.Process(target=_pipe_worker, args=(r, world, path, T, q)) for r in range(world)]
    for pr in ps:
        pr.start()
    loss_k, grads_k, segs = q.get(timeout=300)
    for pr in ps:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    torch.manual_seed(0)
    fwd_fn, bwd_fn = D.lif_segment_fns(snn.LIFParams.paper(), spike_fmt="io")
    model = torch.nn.Sequential(
        P.TimeFolded(torch.nn.Conv2d(2, 16, 3, padding=1)),
        P.TimeSplitLIFLayer(0, 1, None, fwd_fn, bwd_fn, n_chunks=2),
        P.TimeFolded(torch.nn.Flatten()), P.TimeFolded(torch.nn.Linear(16 * 16 * 16, 10))).cuda()
    x = snn_synth.normal_tensor(93, T, 4 * 2 * 16 * 16, device="cuda").reshape(T, 4, 2, 16, 16)
    loss_1 = P.TimeSplitTrainer(model, T).step(x, torch.nn.functional.cross_entropy,
                                               torch.arange(4, device="cuda") % 10)
    assert loss_k == pytest.approx(float(loss_1), rel=1e-5)
    for gk, p in zip(grads_k, model.parameters()):
        np.testing.assert_allclose(gk, p.grad.cpu().numpy(), rtol=2e-4, atol=2e-5)
    # The time-split LIF layer inside the k-rank training step, anchored to the oracle: on its
    # own (conv-produced) input and incoming gradient, the spikes and dL/dX the k ranks
    # produced together equal the fp64 oracle's whole-axis answer.
    from parity import oracle_check
    cat = lambda i: torch.from_numpy(np.concatenate([sg[i] for sg in segs], 0))
    rep = oracle_check(snn.LIFParams.paper(), cat(1), cat(3), cat(2), cat(4))
    assert rep.ok, str(rep)
