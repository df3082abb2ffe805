"""The time split behind the C ABI (include/snn_lif.h snn_comm_* / snn_lif_*_tsplit): chunked
fused kernels with the boundary V / dL/dV moved by NCCL send/recv (
PAPER.md:245-259).

* One rank (a 1-process NCCL communicator): the chunked launches over column windows of the
  layer equal one whole-axis call bitwise and the oracle.
* Two ranks on this single GPU: NCCL refuses two ranks on one device ("duplicate GPU"), so
  each process gets its own NCCL_HOSTID and the ranks talk over the socket transport on
  loopback -- the same snn_lif_*_tsplit code path a multi-GPU box runs over NVLink, checked
  bitwise against k = 1 and against the oracle."""
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
import snn_synth  # noqa: E402
from parity import oracle_check  # noqa: E402

PAPER = snn.LIFParams.paper()


@pytest.fixture(scope="module")
def comm1():
    c = D.NcclComm()          # no process group: a 1-rank communicator
    yield c
    c.close()


@pytest.mark.parametrize("T,N,n_chunks", [(40, 5000, 3), (17, 4096, 1), (33, 12288, 7), (16, 5001, 4)])
@pytest.mark.parametrize("spike_fmt,save_mode", [("u8", "recompute"), ("bits", "h"), ("io", "recompute")])
def test_single_rank_tsplit_equals_whole_and_oracle(comm1, T, N, n_chunks, spike_fmt, save_mode):
    X = snn_synth.normal_tensor(1234, T, N, device="cuda")
    G = snn_synth.normal_tensor(4321, T, N, device="cuda")
    v0 = snn_synth.normal_tensor(1235, 1, N, std=0.5)[0].cuda()
    gvf = snn_synth.normal_tensor(4322, 1, N)[0].cuda()
    f = D.lif_forward_tsplit(comm1, X, PAPER, n_chunks=n_chunks, spike_fmt=spike_fmt, save_mode=save_mode,
                             v_init=v0)
    gx, gvi = D.lif_backward_tsplit(comm1, G, f, n_chunks=n_chunks, grad_v_final=gvf)
    w = snn.lif_forward(X, PAPER, v_init=v0, spike_fmt=spike_fmt, save_mode=save_mode)
    gw, gviw = snn.lif_backward(G, w, grad_v_final=gvf)
    torch.cuda.synchronize()
    assert torch.equal(f.spikes, w.spikes) and torch.equal(f.v_final, w.v_final)
    assert torch.equal(gx, gw) and torch.equal(gvi, gviw)
    S = f.spikes if spike_fmt != "bits" else snn.unpack_bits(f.spikes, N)
    rep = oracle_check(PAPER, X.cpu(), G.cpu(), S.cpu(), gx.cpu(), vf_gpu=f.v_final.cpu(), gvi_gpu=gvi.cpu(),
                       v0=v0.cpu(), gvf=gvf.cpu())
    assert rep.ok, str(rep)


def test_tsplit_validation_errors(comm1):
    X = torch.zeros(8, 1024, device="cuda")
    with pytest.raises(RuntimeError, match="INVALID_VALUE"):
        D.lif_forward_tsplit(comm1, X, PAPER, n_chunks=0)
    with pytest.raises(RuntimeError, match="INVALID_VALUE"):
        D.lif_forward_tsplit(comm1, X, snn.LIFParams(tau=0.5))


def test_window_handoff_single_rank_equals_plain_and_oracle(comm1):
    """SURVEY 8(f) f1 over NCCL symmetric windows (snn_handoff_window_*): a 1-rank
    communicator registers its window (ncclMemAlloc + ncclCommWindowRegister), has no time
    neighbour, and its handoff calls are the plain fused kernels -- bitwise equal to
    snn_lif_forward / snn_lif_backward and to the oracle, over two epochs."""
    from paper_2408_00280_b200 import handoff as HO
    T, N = 24, 4099
    X = snn_synth.normal_tensor(1234, T, N, device="cuda")
    G = snn_synth.normal_tensor(4321, T, N, device="cuda")
    w = HO.WindowHandoff(comm1, N)
    try:
        assert w.pointer(0) != 0 and w.pointer(-1) == 0 and w.pointer(1) == 0
        for epoch in (1, 2):
            hf, hb = w.forward_handoff(), w.backward_handoff()
            assert hf.epoch == epoch and hb.epoch == epoch
            assert not any((hf.recv_state, hf.send_state, hb.recv_state, hb.send_state))
            f = HO.lif_forward_handoff(X, PAPER, hf)
            gx, gvi = HO.lif_backward_handoff(G, f, hb)
            ref = snn.lif_forward(X, PAPER)
            gref, gviref = snn.lif_backward(G, ref)
            torch.cuda.synchronize()
            assert torch.equal(f.spikes, ref.spikes) and torch.equal(f.v_final, ref.v_final)
            assert torch.equal(gx, gref) and torch.equal(gvi, gviref)
        rep = oracle_check(PAPER, X.cpu(), G.cpu(), f.spikes.cpu(), gx.cpu(), vf_gpu=f.v_final.cpu(),
                           gvi_gpu=gvi.cpu())
        assert rep.ok, str(rep)
    finally:
        w.close()


# ------------------------------------------------------------------ two ranks, one GPU

def _rendezvous_file():
    import tempfile
    fd, path = tempfile.mkstemp(prefix="snn_pg_")
    os.close(fd)
    os.remove(path)
    return path


def _worker(rank, world, path, T, N, n_chunks, out):
    # distinct host ids: NCCL then treats the two processes as two hosts (no duplicate-GPU
    # refusal) and connects them through its socket transport on loopback
    os.environ.update(NCCL_HOSTID=f"snn-test-host-{rank}", NCCL_P2P_DISABLE="1", NCCL_SHM_DISABLE="1",
                      NCCL_IB_DISABLE="1", NCCL_NET="Socket", NCCL_SOCKET_IFNAME="lo", NCCL_NVLS_ENABLE="0")
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2408_00280_b200 as snn
    from paper_2408_00280_b200 import dist as D
    import snn_synth
    try:
        comm = D.NcclComm()
    except RuntimeError as e:                  # report (the parent kills a peer left waiting)
        out.put(("error", f"rank {rank}: {e}"))
        return
    # the window handoff needs load/store peers: two "hosts" (one per NCCL_HOSTID) are not an
    # LSA team, so creation must refuse cleanly (SNN_ERR_UNSUPPORTED), not hang or fault
    from paper_2408_00280_b200 import handoff as HO
    try:
        HO.WindowHandoff(comm, N).close()
        refusal = "created"
    except RuntimeError as e:
        refusal = str(e)
    p = snn.LIFParams.paper()
    a, b = D.partition_time(T, world)[rank]
    X = snn_synth.normal_tensor(1234, b - a, N, t_offset=a, device="cuda")
    G = snn_synth.normal_tensor(4321, b - a, N, t_offset=a, device="cuda")
    res = []
    for ep in range(2):                        # twice: buffers and events reused
        ts = D.TimeSplitLIF(rank, world, comm, n_chunks=n_chunks, params=p)   # the C ABI path
        spikes, state, vf = ts.forward(X)
        gx, gvi = ts.backward(G, state)
        torch.cuda.synchronize()
        res.append((spikes.cpu().numpy(), gx.cpu().numpy(), None if vf is None else vf.cpu().numpy(),
                    None if gvi is None else gvi.cpu().numpy(), ts.messages_sent))
    comm.close()
    objs = [None] * world
    dist.all_gather_object(objs, (a, b, res, refusal))
    if rank == 0:
        out.put(("ok", objs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_chunks", [(2, 4)])
def test_two_rank_nccl_tsplit_on_one_gpu(world, n_chunks):
    T, N = 48, 8192
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    path = _rendezvous_file()
    ps = [ctx.Process(target=_worker, args=(r, world, path, T, N, n_chunks, q), daemon=True) for r in range(world)]
    for p_ in ps:
        p_.start()
    try:
        status, objs = q.get(timeout=420)
        for p_ in ps:
            p_.join(timeout=60)
    finally:
        for p_ in ps:
            if p_.is_alive():
                p_.kill()
    if status == "error":
        pytest.skip(f"NCCL would not form a 2-rank communicator on one GPU here: {objs}")
    for p_ in ps:
        assert p_.exitcode == 0
    objs = sorted(objs, key=lambda o: o[0])
    X = snn_synth.normal_tensor(1234, T, N, device="cuda")
    G = snn_synth.normal_tensor(4321, T, N, device="cuda")
    f = snn.lif_forward(X, PAPER)
    gx, gvi = snn.lif_backward(G, f)
    torch.cuda.synchronize()
    for e in range(2):
        S = np.concatenate([o[2][e][0] for o in objs])
        GX = np.concatenate([o[2][e][1] for o in objs])
        assert np.array_equal(S, f.spikes.cpu().numpy())          # bitwise = k = 1
        assert np.array_equal(GX, gx.cpu().numpy())
        assert np.array_equal(objs[-1][2][e][2], f.v_final.cpu().numpy())
        assert np.array_equal(objs[0][2][e][3], gvi.cpu().numpy())
    rep = oracle_check(PAPER, X.cpu(), G.cpu(), torch.from_numpy(S), torch.from_numpy(GX),
                       vf_gpu=torch.from_numpy(objs[-1][2][1][2]), gvi_gpu=torch.from_numpy(objs[0][2][1][3]))
    assert rep.ok, str(rep)
    for o in objs:
        assert "UNSUPPORTED" in o[3] and "load/store peer" in o[3], o[3]
    # one message per chunk per boundary per direction
    n_eff = len(D.neuron_chunks(N, n_chunks, 512))
    assert objs[0][2][0][4] == n_eff and objs[-1][2][0][4] == n_eff
