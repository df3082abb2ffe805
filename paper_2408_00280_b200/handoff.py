"""Time-segment split with the boundary handoff fused into the kernels.

PAPER.md:245-255: rank d owns time steps [t_d, t_{d+1}) of every neuron of a layer; the
boundary membrane state flows forward in time (d -> d+1) and dL/dV backward (d+1 -> d).
``dist.TimeSplitLIF`` moves the boundary with NCCL send/recv between per-chunk kernel
launches.  Here there is no separate collective: each rank's fused kernel stores every
tile's carry-out straight into the neighbour's buffer through a peer-mapped pointer and
releases a per-tile flag; the neighbour's kernel waits on that flag at tile start
(include/snn_lif.h ``snn_lif_forward_handoff``).  One launch per rank per direction; the
wavefront lag between ranks is one tile.

Buffers (per rank, per direction): recv_state [N] fp32, recv_ready / send_ack flags
[ceil(N/256)] int32, allocated with cudaMalloc so their CUDA IPC handles map the whole
allocation.  ``PeerHandoff`` exchanges the handles over a torch.distributed group (gloo
or NCCL) and opens the neighbours' buffers (cudaIpcOpenMemHandle: NVLink peer mappings
on a multi-GPU box; the same device works too, which the tests use).  ``WindowHandoff``
takes the buffers and peer mappings from the NCCL communicator of the time split instead
(symmetric memory windows).
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch
import torch.distributed as dist

from . import _lib
from .lif import (LIFForward, LIFParams, _check_2d, _like_x, _ptr, _stream, _vec, alloc_spikes,
                  make_shape)

_cudart = None


def cudart():
    global _cudart
    if _cudart is None:
        torch.cuda.init()
        _cudart = ctypes.CDLL("libcudart.so.12")
        _cudart.cudaMalloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t]
        _cudart.cudaFree.argtypes = [ctypes.c_void_p]
        _cudart.cudaMemset.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t]
        _cudart.cudaIpcGetMemHandle.argtypes = [ctypes.POINTER(_IpcHandle), ctypes.c_void_p]
        _cudart.cudaIpcOpenMemHandle.argtypes = [ctypes.POINTER(ctypes.c_void_p), _IpcHandle,
                                                 ctypes.c_uint]
        _cudart.cudaIpcCloseMemHandle.argtypes = [ctypes.c_void_p]
    return _cudart


class _IpcHandle(ctypes.Structure):
    _fields_ = [("reserved", ctypes.c_char * 64)]


def _check(err, what):
    if err != 0:
        raise RuntimeError(f"{what} failed with cudaError {err}")


class DeviceBuffer:
    """A cudaMalloc allocation (its IPC handle maps the whole buffer at offset 0)."""

    def __init__(self, nbytes: int):
        self.nbytes = nbytes
        self.ptr = ctypes.c_void_p()
        _check(cudart().cudaMalloc(ctypes.byref(self.ptr), max(nbytes, 256)), "cudaMalloc")
        _check(cudart().cudaMemset(self.ptr, 0, max(nbytes, 256)), "cudaMemset")

    @property
    def addr(self) -> int:
        return self.ptr.value

    def ipc_handle(self) -> bytes:
        h = _IpcHandle()
        _check(cudart().cudaIpcGetMemHandle(ctypes.byref(h), self.ptr), "cudaIpcGetMemHandle")
        return ctypes.string_at(ctypes.addressof(h), 64)   # all 64 bytes (h.reserved stops at NUL)

    def free(self):
        if self.ptr.value:
            cudart().cudaFree(self.ptr)
            self.ptr = ctypes.c_void_p()


def open_ipc(handle: bytes) -> int:
    h = _IpcHandle()
    ctypes.memmove(ctypes.addressof(h), handle, 64)
    p = ctypes.c_void_p()
    _check(cudart().cudaIpcOpenMemHandle(ctypes.byref(p), h, 1), "cudaIpcOpenMemHandle")
    return p.value


class Direction:
    """One rank's receive side of one direction: state + ready flags + ack flags for what
    it sends in that direction."""

    def __init__(self, N: int):
        nblk = _lib.lib.snn_lif_handoff_blocks(N)
        self.recv_state = DeviceBuffer(4 * N)
        self.recv_ready = DeviceBuffer(4 * nblk)
        self.send_ack = DeviceBuffer(4 * nblk)

    def buffers(self):
        return (self.recv_state, self.recv_ready, self.send_ack)

    def free(self):
        for b in self.buffers():
            b.free()


def make_handoff(epoch: int, *, recv=None, send=None) -> "_lib.snn_lif_handoff":
    """recv = (recv_state, recv_ready, recv_ack_peer) addresses of the receive side (or
    None for the first segment); send = (send_state_peer, send_ready_peer, send_ack)."""
    h = _lib.snn_lif_handoff()
    if recv is not None:
        h.recv_state, h.recv_ready, h.recv_ack = recv
    if send is not None:
        h.send_state, h.send_ready, h.send_ack = send
    h.epoch = epoch
    return h


class PeerHandoff:
    """Boundary buffers of this rank + peer mappings of its neighbours, for one layer
    shape (N neurons).  Collective over `group`: every rank constructs it."""

    def __init__(self, N: int, group=None):
        self.N = N
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.fwd = Direction(N)      # receives V from rank-1; acks what it sends to rank+1
        self.bwd = Direction(N)      # receives dL/dV from rank+1; acks what it sends to rank-1
        mine = {k: [b.ipc_handle() for b in d.buffers()] for k, d in (("fwd", self.fwd), ("bwd", self.bwd))}
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self._opened = []

        def peer(r, direction, i):
            addr = open_ipc(allh[r][direction][i])
            self._opened.append(addr)
            return addr

        r, w = self.rank, self.world
        # forward: send to r+1 (its fwd recv_state / recv_ready), my fwd.send_ack collects acks;
        #          receive from r-1, acking into r-1's fwd.send_ack.
        self.f_send = ((peer(r + 1, "fwd", 0), peer(r + 1, "fwd", 1), self.fwd.send_ack.addr)
                       if r + 1 < w else None)
        self.f_recv = ((self.fwd.recv_state.addr, self.fwd.recv_ready.addr, peer(r - 1, "fwd", 2))
                       if r > 0 else None)
        # backward: send to r-1 (its bwd recv_*), receive from r+1 acking into r+1's bwd.send_ack.
        self.b_send = ((peer(r - 1, "bwd", 0), peer(r - 1, "bwd", 1), self.bwd.send_ack.addr)
                       if r > 0 else None)
        self.b_recv = ((self.bwd.recv_state.addr, self.bwd.recv_ready.addr, peer(r + 1, "bwd", 2))
                       if r + 1 < w else None)
        self.f_epoch = 0
        self.b_epoch = 0
        # cudaMemset is asynchronous: without this a peer could publish its first flag into
        # a buffer whose zeroing is still queued here, and the zeroing would then erase it.
        _check(cudart().cudaDeviceSynchronize(), "cudaDeviceSynchronize")
        dist.barrier(group=group)   # every buffer zeroed and mapped before anyone sends

    def forward_handoff(self):
        self.f_epoch += 1
        return make_handoff(self.f_epoch, recv=self.f_recv, send=self.f_send)

    def backward_handoff(self):
        self.b_epoch += 1
        return make_handoff(self.b_epoch, recv=self.b_recv, send=self.b_send)

    def close(self, group=None):
        torch.cuda.synchronize()
        dist.barrier(group=group)
        for a in self._opened:
            cudart().cudaIpcCloseMemHandle(ctypes.c_void_p(a))
        self._opened = []
        dist.barrier(group=group)
        self.fwd.free()
        self.bwd.free()


class WindowHandoff:
    """The same boundary buffers and neighbour pointers as ``PeerHandoff``, taken from an
    NCCL communicator instead of CUDA IPC (include/snn_lif.h snn_handoff_window_*): every
    rank's receive buffers live in one ncclMemAlloc allocation registered as a symmetric
    window on ``comm`` (a ``dist.NcclComm``, rank order = time order), and the neighbours'
    buffers are addressed through the window's LSA mapping (NVLink peers of one node).  Raises
    RuntimeError (SNN_ERR_UNSUPPORTED) when a time neighbour is not a load/store peer.
    Collective: every rank constructs it with the same N."""

    def __init__(self, comm, N: int):
        self.comm = comm
        self.N = N
        self.rank, self.world = comm.rank, comm.world
        self.handle = _lib.snn_handoff_window_create(comm.handle, N)

    def forward_handoff(self):
        return _lib.snn_handoff_window_next(self.handle, 0)

    def backward_handoff(self):
        return _lib.snn_handoff_window_next(self.handle, 1)

    def pointer(self, which: int) -> int:
        """Base address of this rank's buffer (0) or its neighbour's (-1 / +1) as mapped here."""
        return _lib.snn_handoff_window_pointer(self.handle, which)

    def close(self, group=None):
        if getattr(self, "handle", None):
            _lib.snn_handoff_window_destroy(self.handle)
            self.handle = None


def lif_forward_handoff(x: torch.Tensor, params: LIFParams, handoff, *, spike_fmt: str = "u8",
                        save_mode: str = "recompute", v_init: Optional[torch.Tensor] = None,
                        return_v_final: bool = True) -> LIFForward:
    """The local time segment's fused forward; the boundary V arrives / leaves through
    `handoff` inside the kernel (snn_lif_forward_handoff)."""
    _check_2d("x", x)
    T, N = x.shape
    shape = make_shape(x, spike_fmt, save_mode)
    cp = params.to_c()
    v_init = _vec("v_init", v_init, N, x.device)
    spikes = alloc_spikes(x, spike_fmt, shape.ld)   # row stride ld, like x (a column view is fine)
    saved = torch.empty(_lib.snn_lif_saved_bytes(cp, shape) // 4, dtype=torch.float32, device=x.device)
    v_final = torch.empty(N, dtype=torch.float32, device=x.device) if return_v_final else None
    _lib.snn_lif_forward_handoff(cp, shape, _ptr(x), _ptr(v_init), handoff, _ptr(spikes), _ptr(saved),
                                 _ptr(v_final), _stream())
    return LIFForward(spikes, saved, v_final, x, v_init, params, shape)


def lif_backward_handoff(grad_spikes: torch.Tensor, fwd: LIFForward, handoff, *,
                         grad_v_final: Optional[torch.Tensor] = None, return_grad_v_init: bool = True):
    """The local segment's fused backward; dL/dV arrives from the later segment and the
    segment's grad_v_init leaves to the earlier one through `handoff`."""
    x = fwd.x
    T, N = x.shape
    ld = fwd.shape.ld
    grad_spikes = _like_x("grad_spikes", grad_spikes, x, ld)        # every operand walks rows of stride ld
    grad_x = torch.empty((T, ld), dtype=x.dtype, device=x.device)[:, :N]
    grad_v_final = _vec("grad_v_final", grad_v_final, N, x.device)
    gvi = torch.empty(N, dtype=torch.float32, device=x.device) if return_grad_v_init else None
    _lib.snn_lif_backward_handoff(fwd.params.to_c(), fwd.shape, _ptr(grad_spikes),
                                  _ptr(x), _ptr(fwd.saved), _ptr(grad_v_final), handoff,
                                  _ptr(grad_x), _ptr(gvi), _stream())
    return grad_x, gvi
