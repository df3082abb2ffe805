"""The fused boundary handoff: time segments whose kernels exchange the
boundary V / dL/dV through flags + peer stores inside the kernel must be BITWISE equal
to one whole-axis run (the handoff carries exactly the register state)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_00280_b200 as snn  # noqa: E402
from paper_2408_00280_b200 import dist as D  # noqa: E402
from paper_2408_00280_b200 import handoff as HO  # noqa: E402
import snn_synth  # noqa: E402
from parity import oracle_check  # noqa: E402


def _local_dirs(k, N):
    """Per-segment buffers in ONE process (the 'peer' pointers are local addresses)."""
    nblk = snn._lib.lib.snn_lif_handoff_blocks(N)
    mk = lambda: dict(state=torch.zeros(N, device="cuda"),
                      ready=torch.zeros(nblk, dtype=torch.int32, device="cuda"),
                      ack=torch.zeros(nblk, dtype=torch.int32, device="cuda"))
    return [mk() for _ in range(k)], [mk() for _ in range(k)]


def _fwd_h(fd, d, k, epoch):
    recv = (fd[d]["state"].data_ptr(), fd[d]["ready"].data_ptr(), fd[d - 1]["ack"].data_ptr()) if d > 0 else None
    send = (fd[d + 1]["state"].data_ptr(), fd[d + 1]["ready"].data_ptr(), fd[d]["ack"].data_ptr()) if d + 1 < k else None
    return HO.make_handoff(epoch, recv=recv, send=send)


def _bwd_h(bd, d, k, epoch):
    recv = (bd[d]["state"].data_ptr(), bd[d]["ready"].data_ptr(), bd[d + 1]["ack"].data_ptr()) if d + 1 < k else None
    send = (bd[d - 1]["state"].data_ptr(), bd[d - 1]["ready"].data_ptr(), bd[d]["ack"].data_ptr()) if d > 0 else None
    return HO.make_handoff(epoch, recv=recv, send=send)


@pytest.mark.parametrize("k,T,N,dtype,save_mode", [
    (2, 40, 4096, torch.float32, "recompute"),
    (3, 70, 5000, torch.float32, "h"),          # ragged last tile
    (4, 64, 6144, torch.bfloat16, "recompute"),
])
def test_handoff_segments_in_one_process_bitwise(k, T, N, dtype, save_mode):
    """Segments launched in time order on one stream (each completes before the next
    starts), two epochs to exercise the acknowledgement flags."""
    p = snn.LIFParams.paper()
    X = snn_synth.normal_tensor(61, T, N, dtype=dtype, device="cuda")
    G = snn_synth.normal_tensor(62, T, N, dtype=dtype, device="cuda")
    f = snn.lif_forward(X, p, save_mode=save_mode)
    gx_ref, gvi_ref = snn.lif_backward(G, f)
    segs = D.partition_time(T, k)
    fd, bd = _local_dirs(k, N)
    for epoch in (1, 2):
        fwds = []
        for d, (a, b) in enumerate(segs):
            fwds.append(HO.lif_forward_handoff(X[a:b], p, _fwd_h(fd, d, k, epoch), save_mode=save_mode))
        gxs = [None] * k
        gvi = None
        for d in range(k - 1, -1, -1):
            a, b = segs[d]
            gxs[d], g = HO.lif_backward_handoff(G[a:b], fwds[d], _bwd_h(bd, d, k, epoch))
            if d == 0:
                gvi = g
        torch.cuda.synchronize()
        assert torch.equal(torch.cat([q.spikes for q in fwds]), f.spikes)
        assert torch.equal(fwds[-1].v_final, f.v_final)
        assert torch.equal(torch.cat(gxs), gx_ref)
        assert torch.equal(gvi, gvi_ref)
        # flags carry the epoch for every block
        assert int(fd[1]["ready"].min()) == epoch and int(bd[0]["ready"].min()) == epoch
    # anchored to the oracle directly: the k-segment handoff result vs the fp64 oracle
    rep = oracle_check(p, snn_synth.normal_tensor(61, T, N, dtype=dtype), snn_synth.normal_tensor(62, T, N, dtype=dtype),
                       torch.cat([q.spikes for q in fwds]).cpu(), torch.cat(gxs).cpu(),
                       vf_gpu=fwds[-1].v_final.cpu(), gvi_gpu=gvi.cpu(), io_bf16=dtype == torch.bfloat16)
    assert rep.ok, str(rep)


def test_handoff_concurrent_streams_bitwise():
    """Sender and receiver kernels resident at the same time (receiver launched second on
    another stream): the receiver's tiles wait on the sender's per-tile flags."""
    p = snn.LIFParams.paper()
    T, N = 32, 1 << 14
    X = snn_synth.normal_tensor(71, T, N, device="cuda")
    G = snn_synth.normal_tensor(72, T, N, device="cuda")
    f = snn.lif_forward(X, p)
    gx_ref, gvi_ref = snn.lif_backward(G, f)
    fd, bd = _local_dirs(2, N)
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s0):
        f0 = HO.lif_forward_handoff(X[:16], p, _fwd_h(fd, 0, 2, 1))
    with torch.cuda.stream(s1):
        f1 = HO.lif_forward_handoff(X[16:], p, _fwd_h(fd, 1, 2, 1))
        g1, _ = HO.lif_backward_handoff(G[16:], f1, _bwd_h(bd, 1, 2, 1))
    s1.synchronize()
    with torch.cuda.stream(s0):
        g0, gvi = HO.lif_backward_handoff(G[:16], f0, _bwd_h(bd, 0, 2, 1))
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([f0.spikes, f1.spikes]), f.spikes)
    assert torch.equal(torch.cat([g0, g1]), gx_ref) and torch.equal(gvi, gvi_ref)
    rep = oracle_check(p, snn_synth.normal_tensor(71, T, N), snn_synth.normal_tensor(72, T, N),
                       torch.cat([f0.spikes, f1.spikes]).cpu(), torch.cat([g0, g1]).cpu(),
                       vf_gpu=f1.v_final.cpu(), gvi_gpu=gvi.cpu())
    assert rep.ok, str(rep)


@pytest.mark.parametrize("N,view", [(4099, False), (3, False), (2050, True)])
def test_handoff_ragged_and_unaligned_rows(N, view):
    """The fused handoff on shapes the round-1 TMA path refused: a ragged N (odd row stride:
    1-D tensor maps, element-wise stores) and an unaligned column view x[:, 1:] of a wider
    tensor.  Bitwise = whole axis, and = the oracle."""
    p = snn.LIFParams.paper()
    T, k = 40, 2
    Xw = snn_synth.normal_tensor(91, T, N + 1 if view else N, device="cuda")
    Gw = snn_synth.normal_tensor(92, T, N + 1 if view else N, device="cuda")
    X, G = (Xw[:, 1:], Gw[:, 1:]) if view else (Xw, Gw)
    f = snn.lif_forward(X, p)
    gx_ref, gvi_ref = snn.lif_backward(G, f)
    segs = D.partition_time(T, k)
    fd, bd = _local_dirs(k, N)
    fwds = [HO.lif_forward_handoff(X[a:b], p, _fwd_h(fd, d, k, 1)) for d, (a, b) in enumerate(segs)]
    g1, _ = HO.lif_backward_handoff(G[segs[1][0]:], fwds[1], _bwd_h(bd, 1, k, 1))
    g0, gvi = HO.lif_backward_handoff(G[: segs[0][1]], fwds[0], _bwd_h(bd, 0, k, 1))
    torch.cuda.synchronize()
    S = torch.cat([q.spikes for q in fwds])
    assert torch.equal(S, f.spikes) and torch.equal(fwds[-1].v_final, f.v_final)
    assert torch.equal(torch.cat([g0, g1]), gx_ref) and torch.equal(gvi, gvi_ref)
    rep = oracle_check(p, X.cpu(), G.cpu(), S.cpu(), torch.cat([g0, g1]).cpu(), vf_gpu=fwds[-1].v_final.cpu(),
                       gvi_gpu=gvi.cpu())
    assert rep.ok, str(rep)


# ------------------------------------------------------------------ k processes, CUDA IPC

def _rendezvous_file():
    import tempfile
    fd, path = tempfile.mkstemp(prefix="snn_pg_")
    os.close(fd)
    os.remove(path)
    return path


def _ipc_worker(rank, world, path, T, N, out):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2408_00280_b200 as snn
    from paper_2408_00280_b200 import dist as D
    from paper_2408_00280_b200 import handoff as HO
    import snn_synth
    p = snn.LIFParams.paper()
    a, b = D.partition_time(T, world)[rank]
    X = snn_synth.normal_tensor(81, b - a, N, t_offset=a, device="cuda")
    G = snn_synth.normal_tensor(82, b - a, N, t_offset=a, device="cuda")
    ph = HO.PeerHandoff(N)
    res = []
    for _ in range(2):                      # two epochs: acknowledgement flags in use
        f = HO.lif_forward_handoff(X, p, ph.forward_handoff())
        gx, gvi = HO.lif_backward_handoff(G, f, ph.backward_handoff())
        torch.cuda.synchronize()
        res.append((f.spikes.cpu().numpy(), gx.cpu().numpy(), f.v_final.cpu().numpy(), gvi.cpu().numpy()))
        dist.barrier()
    ph.close()
    objs = [None] * world
    dist.all_gather_object(objs, (a, b, res))
    if rank == 0:
        out.put(objs)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_handoff_ipc_processes_bitwise(world):
    """k processes on one GPU, each mapping its neighbours' buffers with CUDA IPC (the
    same calls map NVLink peers on a multi-GPU box)."""
    T, N = 48, 4096
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    path = _rendezvous_file()
    ps = [ctx.Process(target=_ipc_worker, args=(r, world, path, T, N, q)) for r in range(world)]
    for pr in ps:
        pr.start()
    objs = sorted(q.get(timeout=300), key=lambda o: o[0])
    for pr in ps:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = snn.LIFParams.paper()
    X = snn_synth.normal_tensor(81, T, N, device="cuda")
    G = snn_synth.normal_tensor(82, T, N, device="cuda")
    f = snn.lif_forward(X, p)
    gx, gvi = snn.lif_backward(G, f)
    torch.cuda.synchronize()
    rep = oracle_check(p, snn_synth.normal_tensor(81, T, N), snn_synth.normal_tensor(82, T, N),
                       torch.from_numpy(np.concatenate([o[2][1][0] for o in objs])),
                       torch.from_numpy(np.concatenate([o[2][1][1] for o in objs])),
                       vf_gpu=torch.from_numpy(objs[-1][2][1][2]), gvi_gpu=torch.from_numpy(objs[0][2][1][3]))
    assert rep.ok, str(rep)
    for e in range(2):
        assert np.array_equal(np.concatenate([o[2][e][0] for o in objs]), f.spikes.cpu().numpy())
        assert np.array_equal(np.concatenate([o[2][e][1] for o in objs]), gx.cpu().numpy())
        assert np.array_equal(objs[-1][2][e][2], f.v_final.cpu().numpy())
        assert np.array_equal(objs[0][2][e][3], gvi.cpu().numpy())
