"""Multi-GPU partitioning of the fused LIF path.

Two ways the path shards on one 8xB200 box:

1. Neuron / batch sharding (``shard_range``): every neuron's recurrence is autonomous
   (PAPER.md:191-193), so rank r owns a contiguous neuron range and there is no
   collective on the data path -- bench.py's weak-scaling runs and BASELINE configs[4].
2. The paper's time-segment split (``TimeSplitLIF``; Fig. 1(b)):
   rank d owns time steps [t_d, t_{d+1}) of every neuron (``partition_time``, the SPEC
   remainder rule).  Forward: receive the post-reset V of the previous
   segment, run the fused forward on the local segment, send the final V to d+1.
   Backward: receive dL/dV from d+1, run the fused backward, send grad_v_init to d-1.
   The payload is the [N] fp32 boundary state.  To give the k ranks
   concurrent work on one layer the neurons are cut into M chunks processed
   in the same order on every rank: rank d starts chunk m as soon as chunk m's boundary
   arrives, a wavefront whose fill costs (k-1)/(M+k-1).

Segmented execution is bitwise equal to the whole axis (the kernels carry exactly the
state a whole run keeps in registers, tests/test_gpu_parity.py), so the
time split is bitwise equal to k = 1.

The host orchestration is transport-agnostic: ``NcclTransport`` moves device tensors
with torch.distributed point-to-point ops (NCCL over NVLink on the GPU box);
``HostTransport`` stages through pinned host memory with gloo, which lets the same
protocol be tested with several processes on one GPU or on CPU (tests/test_dist.py).
The per-segment compute is a callable, so the CPU tests can drive the protocol with the
oracle; the product path passes the CUDA kernels (``lif_segment_forward`` / backward).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


# ----------------------------------------------------------------------------- partitions

def partition_time(T: int, k: int) -> List[Tuple[int, int]]:
    """k contiguous near-equal segments of [0, T); the first T mod k get one extra step
    (SURVEY R17).  Raises for k < 1 or k > T."""
    if k < 1 or k > T:
        raise ValueError(f"need 1 <= k <= T (k={k}, T={T})")
    q, r = divmod(T, k)
    out, t = [], 0
    for d in range(k):
        n = q + (1 if d < r else 0)
        out.append((t, t + n))
        t += n
    return out


def shard_range(N: int, world: int, rank: int, align: int = 1) -> Tuple[int, int]:
    """Contiguous neuron range of `rank` (boundaries multiples of `align` except the end)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    units = -(-N // align)
    q, r = divmod(units, world)
    lo = rank * q + min(rank, r)
    hi = lo + q + (1 if rank < r else 0)
    return min(N, lo * align), min(N, hi * align)


def neuron_chunks(N: int, M: int, align: int = 512) -> List[Tuple[int, int]]:
    """M contiguous neuron chunks (boundaries on `align`, the TMA tile width)."""
    M = max(1, min(M, -(-N // align)))
    return [shard_range(N, M, m, align) for m in range(M)]


# ----------------------------------------------------------------------------- Eq. 4-5

def speedup_mu(Ts: float, Tc: float, k: int) -> float:
    """Eq. 5: mu = k T_s / (k (k-1) T_c + T_s)."""
    return k * Ts / (k * (k - 1) * Tc + Ts)


def optimal_k(Ts: float, Tc: float) -> float:
    """Continuous optimum of Eq. 5, k = sqrt(T_s / T_c)."""
    return math.sqrt(Ts / Tc)


def model_curve(ratios: Sequence[float], k_max: int):
    """Fig. 4: rows (ratio, k, mu) with T_c = 1, T_s = ratio."""
    return [(r, k, speedup_mu(r, 1.0, k)) for r in ratios for k in range(1, k_max + 1)]


def pipeline_efficiency(M: int, k: int) -> float:
    """Wavefront efficiency of M neuron chunks over k time segments."""
    return M / (M + k - 1)


# ----------------------------------------------------------------------------- transports

class NcclTransport:
    """Device tensors over torch.distributed P2P (NCCL on NVLink / NVSwitch)."""

    def __init__(self, group=None):
        self.group = group

    def isend(self, t: torch.Tensor, dst: int):
        return dist.isend(t, dst, group=self.group)

    def irecv(self, t: torch.Tensor, src: int):
        return dist.irecv(t, src, group=self.group)


class NcclComm:
    """The C ABI's NCCL communicator (include/snn_lif.h ``snn_comm``) over the ranks of a
    torch.distributed group; rank order is time order.  Rank 0 draws the ncclUniqueId and the
    group broadcasts it (any backend: gloo or NCCL); every rank then joins the communicator
    on its current CUDA device.  Used as the transport of ``TimeSplitLIF`` it runs the whole
    segment -- chunked kernels and NCCL send/recv -- inside ``snn_lif_*_tsplit``."""

    def __init__(self, group=None):
        from . import _lib
        self._lib = _lib
        if dist.is_available() and dist.is_initialized():
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        uid = [_lib.snn_nccl_unique_id() if self.rank == 0 else None]
        if self.world > 1:
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(uid, src=src, group=group)
        self.handle = _lib.snn_comm_create(uid[0], self.world, self.rank)

    def close(self):
        if getattr(self, "handle", None):
            self._lib.snn_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lif_forward_tsplit(comm: NcclComm, x_local: torch.Tensor, params, *, n_chunks: int = 32,
                       spike_fmt: str = "u8", save_mode: str = "recompute",
                       v_init: Optional[torch.Tensor] = None):
    """This rank's time segment of one LIF layer's fused forward, boundary V through NCCL
    (snn_lif_forward_tsplit).  x_local: [T_d, N] CUDA.  Returns a LIFForward whose v_final
    is the layer's final V on the last rank (None elsewhere)."""
    from . import _lib
    from .lif import LIFForward, _check_2d, _ptr, _stream, _vec, alloc_spikes, make_shape, saved_bytes
    _check_2d("x_local", x_local)
    T_d, N = x_local.shape
    shape = make_shape(x_local, spike_fmt, save_mode)
    dev = x_local.device
    spikes = alloc_spikes(x_local, spike_fmt, shape.ld)
    saved = (torch.empty(saved_bytes(params, shape) // 4, dtype=torch.float32, device=dev)
             if save_mode != "none" else None)
    first, last = comm.rank == 0, comm.rank == comm.world - 1
    v_in = _vec("v_init", v_init, N, dev) if first else torch.empty(N, dtype=torch.float32, device=dev)
    v_out = torch.empty(N, dtype=torch.float32, device=dev)
    _lib.snn_lif_forward_tsplit(comm.handle, params.to_c(), shape, int(n_chunks), _ptr(x_local), _ptr(spikes),
                                _ptr(saved), _ptr(v_in), _ptr(v_out), _stream(dev))
    f = LIFForward(spikes, saved, v_out if last else None, x_local, v_in if first else None, params, shape)
    f.v_in_ws = v_in
    return f


def lif_backward_tsplit(comm: NcclComm, grad_local: torch.Tensor, fwd, *, n_chunks: int = 32,
                        grad_v_final: Optional[torch.Tensor] = None, grad_x: Optional[torch.Tensor] = None):
    """This rank's segment of the fused backward, dL/dV through NCCL (snn_lif_backward_tsplit).
    Returns (grad_x [T_d, N], grad_v_init [N] on rank 0 / None elsewhere)."""
    from . import _lib
    from .lif import _like_x, _ptr, _stream, _vec
    x = fwd.x
    T_d, N = x.shape
    dev = x.device
    ld = fwd.shape.ld
    grad_local = _like_x("grad_local", grad_local, x, ld)
    if grad_x is None:
        grad_x = torch.empty((T_d, ld), dtype=x.dtype, device=dev)[:, :N]
    first, last = comm.rank == 0, comm.rank == comm.world - 1
    g_in = _vec("grad_v_final", grad_v_final, N, dev) if last else torch.empty(N, dtype=torch.float32, device=dev)
    g_out = torch.empty(N, dtype=torch.float32, device=dev)
    _lib.snn_lif_backward_tsplit(comm.handle, fwd.params.to_c(), fwd.shape, int(n_chunks), _ptr(grad_local),
                                 _ptr(x), _ptr(getattr(fwd, "v_in_ws", fwd.v_init)), _ptr(fwd.saved),
                                 _ptr(grad_x), _ptr(g_in), _ptr(g_out),
                                 _stream(dev))
    return grad_x, (g_out if first else None)


class HostTransport:
    """Stages through host memory with a CPU-capable backend (gloo).  Used by the tests
    to run the protocol with several processes on one GPU or on CPU; not a hot path."""

    def __init__(self, group=None):
        self.group = group

    class _Req:
        def __init__(self, work, dev_t=None, host_t=None):
            self.work, self.dev_t, self.host_t = work, dev_t, host_t

        def wait(self):
            self.work.wait()
            if self.dev_t is not None:
                self.dev_t.copy_(self.host_t)

    def isend(self, t: torch.Tensor, dst: int):
        h = t.detach().to("cpu").contiguous()
        return self._Req(dist.isend(h, dst, group=self.group))

    def irecv(self, t: torch.Tensor, src: int):
        if t.is_cuda:
            h = torch.empty(t.shape, dtype=t.dtype)
            return self._Req(dist.irecv(h, src, group=self.group), t, h)
        return self._Req(dist.irecv(t, src, group=self.group))


# ----------------------------------------------------------------------------- time split

@dataclass
class SegmentState:
    """What one rank keeps between its forward and backward: per-chunk forward contexts."""
    ctxs: list
    chunks: List[Tuple[int, int]]


class TimeSplitLIF:
    """The paper's time-segment pipeline for one LIF layer.

    ``rank`` (0..k-1) owns time segment ``partition_time(T, k)[rank]``; ranks are ordered
    like time.  ``fwd_fn(x_chunk, v_in) -> (ctx, spikes_chunk, v_out)`` and
    ``bwd_fn(g_chunk, ctx, g_in) -> (gx_chunk, g_out)`` run one segment of one neuron
    chunk (the product passes the fused CUDA kernels, see ``lif_segment_fns``).
    Messages per chunk per direction: exactly one per segment boundary, i.e.
    (k-1) per chunk per layer in total.
    """

    def __init__(self, rank: int, k: int, transport, n_chunks: int = 32, align: int = 512, *,
                 params=None, spike_fmt: str = "u8", save_mode: str = "recompute"):
        """transport: ``NcclComm`` (the product: the C ABI runs the whole segment, chunk kernels
        and NCCL send/recv, in snn_lif_*_tsplit; ``params`` / ``spike_fmt`` / ``save_mode`` then
        configure it), or any object with isend / irecv (NcclTransport, HostTransport) driving the
        per-chunk callables given to forward / backward."""
        self.rank, self.k, self.t = rank, k, transport
        self.n_chunks, self.align = n_chunks, align
        self.params, self.spike_fmt, self.save_mode = params, spike_fmt, save_mode
        self.messages_sent = 0

    def _c_abi(self) -> bool:
        return isinstance(self.t, NcclComm)

    def forward(self, x_local: torch.Tensor, fwd_fn: Optional[Callable] = None, *,
                v_init: Optional[torch.Tensor] = None):
        """x_local: [T_d, N] (this rank's time segment).  Returns (spikes_local [T_d, N], state,
        v_final) -- v_final is the layer's final V on the last rank, else None.

        When ``fwd_fn.writes_into`` is set (the CUDA segment functions), the segment's spikes
        are allocated ONCE here and every chunk writes its column view of them (no per-chunk
        buffers, no concatenation); otherwise the chunk results are concatenated."""
        T_d, N = x_local.shape
        chunks = neuron_chunks(N, self.n_chunks, self.align)
        if self._c_abi():
            f = lif_forward_tsplit(self.t, x_local, self.params, n_chunks=self.n_chunks, spike_fmt=self.spike_fmt,
                                   save_mode=self.save_mode, v_init=v_init)
            self.messages_sent += len(chunks) if self.rank + 1 < self.k else 0
            return f.spikes, SegmentState([f], chunks), f.v_final
        dev = x_local.device
        prev, nxt = self.rank - 1, self.rank + 1
        into = getattr(fwd_fn, "writes_into", False)
        out = fwd_fn.alloc_spikes(x_local) if into else None
        ctxs, spikes, sends = [], [], []
        v_final = torch.empty(N, dtype=torch.float32, device=dev) if nxt >= self.k else None
        for (a, b) in chunks:
            if prev >= 0:
                v_in = torch.empty(b - a, dtype=torch.float32, device=dev)
                self.t.irecv(v_in, prev).wait()
            else:
                v_in = None if v_init is None else v_init[a:b].contiguous()
            if into:
                ctx, spk, v_out = fwd_fn(x_local[:, a:b], v_in, out=out[:, a:b])
            else:
                ctx, spk, v_out = fwd_fn(x_local[:, a:b], v_in)
                spikes.append(spk)
            ctxs.append(ctx)
            if nxt < self.k:
                sends.append(self.t.isend(v_out, nxt))
                self.messages_sent += 1
            else:
                v_final[a:b] = v_out
        for s in sends:
            s.wait()
        if not into:
            out = torch.cat(spikes, dim=1)
        return out, SegmentState(ctxs, chunks), v_final

    def backward(self, g_local: torch.Tensor, state: SegmentState, bwd_fn: Optional[Callable] = None, *,
                 grad_v_final: Optional[torch.Tensor] = None):
        """g_local: [T_d, N] dL/dS of this segment.  Returns (grad_x [T_d, N], grad_v_init) --
        grad_v_init is the layer's dL/dV[-1] on rank 0, else None.  grad_x is allocated once
        when ``bwd_fn.writes_into`` is set (chunks write their column views)."""
        if self._c_abi():
            gx, gvi = lif_backward_tsplit(self.t, g_local, state.ctxs[0], n_chunks=self.n_chunks,
                                          grad_v_final=grad_v_final)
            self.messages_sent += len(state.chunks) if self.rank > 0 else 0
            return gx, gvi
        dev = g_local.device
        T_d, N = g_local.shape
        prev, nxt = self.rank - 1, self.rank + 1
        into = getattr(bwd_fn, "writes_into", False)
        out = torch.empty((T_d, N), dtype=g_local.dtype, device=dev) if into else None
        gxs, sends = [], []
        g_first = torch.empty(N, dtype=torch.float32, device=dev) if prev < 0 else None
        for (a, b), ctx in zip(state.chunks, state.ctxs):
            if nxt < self.k:
                g_in = torch.empty(b - a, dtype=torch.float32, device=dev)
                self.t.irecv(g_in, nxt).wait()
            else:
                g_in = None if grad_v_final is None else grad_v_final[a:b].contiguous()
            if into:
                _, g_out = bwd_fn(g_local[:, a:b], ctx, g_in, out=out[:, a:b])
            else:
                gx, g_out = bwd_fn(g_local[:, a:b], ctx, g_in)
                gxs.append(gx)
            if prev >= 0:
                sends.append(self.t.isend(g_out, prev))
                self.messages_sent += 1
            else:
                g_first[a:b] = g_out
        for s in sends:
            s.wait()
        if not into:
            out = torch.cat(gxs, dim=1)
        return out, g_first


def lif_segment_fns(params, *, spike_fmt: str = "u8", save_mode: str = "recompute"):
    """(fwd_fn, bwd_fn) running one segment of one neuron chunk through the fused CUDA
    kernels (C ABI) -- the per-chunk compute of TimeSplitLIF over a torch.distributed
    transport.  Both write into column views of segment-wide outputs (``writes_into``):
    a chunk view x[:, a:b] has row stride N, and so do the views of the [T_d, N] outputs."""
    from .lif import lif_backward, lif_forward, alloc_spikes

    def fwd_fn(x_chunk, v_in, out=None):
        f = lif_forward(x_chunk, params, v_init=v_in, spike_fmt=spike_fmt, save_mode=save_mode,
                        spikes=out)
        return f, f.spikes, f.v_final

    def bwd_fn(g_chunk, ctx, g_in, out=None):
        return lif_backward(g_chunk, ctx, grad_v_final=g_in, grad_x=out)

    # bit-packed spikes have dense [T, ceil(n/32)] rows per call: no column views
    fwd_fn.writes_into = spike_fmt != "bits"
    fwd_fn.alloc_spikes = lambda x: alloc_spikes(x, spike_fmt)
    bwd_fn.writes_into = True
    return fwd_fn, bwd_fn
