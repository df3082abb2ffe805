"""Layer-pipelined time-split training (the paper's Fig. 1(b),
PAPER.md:150-153 and 245-255).

Every rank owns a contiguous time segment [t_d, t_{d+1}) of EVERY layer of a spiking
network.  Time-independent operators (conv, linear, pooling -- applied to all time steps
of the segment at once, [T_d * B, ...]) need no communication.  Each LIF layer hands its
boundary state to the next rank in the forward (V) and to the previous rank in the
backward (dL/dV) -- ``dist.TimeSplitLIF`` with any transport.  While rank d+1 still waits
for rank d's boundary of layer l, rank d already runs layer l+1: the layer-level overlap
Eq. 4b presumes.  Weight gradients are partial sums over each rank's time
segment, so they are summed across ranks (an all-reduce, like data parallelism over time).

``TimeSplitLIFFunction`` is the autograd glue (the paper's FusedLIF of Listing 1,
PAPER.md:294-302, made segment-aware); ``TimeSplitLIFLayer`` is the module; and
``TimeSplitTrainer`` runs forward, loss, backward and the gradient all-reduce.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

from .dist import TimeSplitLIF


class TimeSplitLIFFunction(torch.autograd.Function):
    """spikes_local = TimeSplitLIFFunction.apply(x_local, ts, fwd_fn, bwd_fn)

    x_local: [T_d, N] (this rank's segment of the layer input, time-major).  fwd_fn /
    bwd_fn: per-chunk segment compute (``dist.lif_segment_fns`` with spike_fmt="io" for the
    CUDA kernels).  The boundary exchange happens inside ts.forward / ts.backward."""

    @staticmethod
    def forward(ctx, x_local, ts: TimeSplitLIF, fwd_fn: Callable, bwd_fn: Callable):
        spikes, state, _ = ts.forward(x_local, fwd_fn)
        ctx.ts, ctx.state, ctx.bwd_fn = ts, state, bwd_fn
        return spikes.to(x_local.dtype)

    @staticmethod
    def backward(ctx, grad_spikes):
        gx, _ = ctx.ts.backward(grad_spikes.contiguous(), ctx.state, ctx.bwd_fn)
        ctx.state = None
        return gx.to(grad_spikes.dtype), None, None, None


class TimeSplitLIFLayer(torch.nn.Module):
    """A LIF layer whose time axis is split across the ranks of a process group.  Input
    [T_d, B, ...]; trailing dims are flattened into the neuron axis."""

    def __init__(self, rank: int, world: int, transport, fwd_fn: Callable, bwd_fn: Callable,
                 n_chunks: int = 4, align: int = 512):
        super().__init__()
        self.ts = TimeSplitLIF(rank, world, transport, n_chunks=n_chunks, align=align)
        self.fwd_fn, self.bwd_fn = fwd_fn, bwd_fn

    def forward(self, x):
        T = x.shape[0]
        y = TimeSplitLIFFunction.apply(x.reshape(T, -1), self.ts, self.fwd_fn, self.bwd_fn)
        return y.reshape(x.shape)


class TimeFolded(torch.nn.Module):
    """Apply a time-independent module to every time step of [T, B, ...] at once."""

    def __init__(self, module: torch.nn.Module):
        super().__init__()
        self.m = module

    def forward(self, x):
        T, B = x.shape[:2]
        y = self.m(x.reshape(T * B, *x.shape[2:]))
        return y.reshape(T, B, *y.shape[1:])


class TimeSplitTrainer:
    """One training step of a time-split network (Fig. 1(b)).

    ``model`` maps this rank's input segment [T_d, B, ...] to per-step outputs
    [T_d, B, classes].  The loss is defined on the time-summed output of the WHOLE axis
    (rate coding): each rank contributes its segment's partial sum, the partial sums are
    all-reduced, and the gradient of the loss w.r.t. each rank's outputs is broadcast
    back -- so the result equals one whole-axis step.  Weight gradients are then
    all-reduced (summed over segments)."""

    def __init__(self, model: torch.nn.Module, T_total: int, group=None):
        self.model, self.T_total, self.group = model, T_total, group

    def step(self, x_local: torch.Tensor, loss_fn: Callable, target: torch.Tensor):
        out = self.model(x_local)                         # [T_d, B, C]
        part = out.sum(dim=0)                             # this segment's share of sum_t out
        total = part.detach().clone()
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(total, group=self.group)
        total.requires_grad_(True)
        rate = total / self.T_total
        loss = loss_fn(rate, target)
        (g_total,) = torch.autograd.grad(loss, total)     # identical on every rank
        part.backward(g_total)                            # through this rank's segment
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            for p in self.model.parameters():
                if p.grad is not None:
                    dist.all_reduce(p.grad, group=self.group)
        return loss.detach()
