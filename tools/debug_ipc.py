"""Debug driver for the IPC handoff: 2 processes on cuda:0, prints progress."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist, torch.multiprocessing as mp


def w(rank, world, path):
    t0 = time.time()
    log = lambda *a: print(f"[r{rank} {time.time()-t0:6.2f}]", *a, flush=True)
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2408_00280_b200 as snn
    from paper_2408_00280_b200 import handoff as HO, dist as D
    import snn_synth
    log("init")
    N, T = int(os.environ.get("DBG_N", 4096)), int(os.environ.get("DBG_T", 48))
    a, b = D.partition_time(T, world)[rank]
    X = snn_synth.normal_tensor(81, b - a, N, t_offset=a, device="cuda")
    ph = HO.PeerHandoff(N)
    log("peer ok", ph.f_send, ph.f_recv)
    for it in range(int(os.environ.get("DBG_IT", 1))):
        f = HO.lif_forward_handoff(X, snn.LIFParams.paper(), ph.forward_handoff())
        log("launched fwd", it)
        torch.cuda.synchronize()
        log("fwd done", it, f.v_final[:2].tolist())
        if os.environ.get("DBG_BWD"):
            G = snn_synth.normal_tensor(82, b - a, N, t_offset=a, device="cuda")
            gx, gvi = HO.lif_backward_handoff(G, f, ph.backward_handoff())
            torch.cuda.synchronize()
            log("bwd done", it, gvi[:2].tolist())
    ph.close()
    log("closed")
    dist.destroy_process_group()


if __name__ == "__main__":
    path = "/tmp/snn_dbg_pg"
    if os.path.exists(path):
        os.remove(path)
    mp.get_context("spawn")
    ps = [mp.get_context("spawn").Process(target=w, args=(r, 2, path)) for r in range(2)]
    [p.start() for p in ps]
    [p.join() for p in ps]
    print("exit", [p.exitcode for p in ps])
