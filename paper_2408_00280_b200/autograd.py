"""The paper's programming model (Listing 1): ``FusedLIF`` is a
``torch.autograd.Function`` whose forward / backward are the fused kernels, and
``LIFLayer`` is the ``nn.Module`` a user drops into ``torch.nn.Sequential(..., LIFLayer(args), ...)``.

Unlike Listing 1 (whose ctx stores only ``args``) the forward keeps what
Eq. 3 needs: the V checkpoints (save_mode "recompute") plus a reference to x, or H
(save_mode "h") -- SURVEY D5 / R13.
"""
from __future__ import annotations

from typing import Optional

import torch

from .lif import (AffineSpec, LIFForward, LIFParams, lif_backward, lif_backward_affine, lif_forward,
                  lif_forward_affine)


class FusedLIF(torch.autograd.Function):
    """spikes = FusedLIF.apply(x, params, v_init, save_mode); x: CUDA [T, N] fp32/bf16.
    Spikes are returned in x's dtype (0/1), the form the next ANN operator consumes."""

    @staticmethod
    def forward(ctx, x: torch.Tensor, params: LIFParams, v_init: Optional[torch.Tensor] = None,
                save_mode: str = "recompute"):
        x = x if x.stride(-1) == 1 else x.contiguous()
        fwd = lif_forward(x, params, v_init=v_init, spike_fmt="io", save_mode=save_mode,
                          return_v_final=False)
        # through save_for_backward (not as attributes of ctx): autograd's version check
        # then catches an in-place edit of x before the RECOMPUTE backward re-reads it, a
        # retained graph can run backward twice, and the output is not kept alive by ctx.
        ctx.save_for_backward(x, fwd.saved, v_init)
        ctx.params, ctx.shape = params, fwd.shape
        ctx.has_v_init = v_init is not None
        return fwd.spikes

    @staticmethod
    def backward(ctx, grad_spikes: torch.Tensor):
        x, saved, v_init = ctx.saved_tensors
        fwd = LIFForward(None, saved, None, x, v_init, ctx.params, ctx.shape)
        gx, gvi = lif_backward(grad_spikes.to(x.dtype), fwd,
                               return_grad_v_init=ctx.has_v_init and ctx.needs_input_grad[2])
        return gx, None, gvi, None


class LIFLayer(torch.nn.Module):
    """Temporally fused LIF layer.  Input [T, ...] (time-major); all
    trailing dims are flattened into the neuron axis N."""

    def __init__(self, params: Optional[LIFParams] = None, save_mode: str = "recompute", **kw):
        super().__init__()
        self.params = params if params is not None else LIFParams(**kw)
        self.save_mode = save_mode

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        T = x.shape[0]
        y = FusedLIF.apply(x.reshape(T, -1), self.params, None, self.save_mode)
        return y.reshape(x.shape)

    def extra_repr(self) -> str:
        return f"{self.params}, save_mode={self.save_mode!r}"


class FusedAffineLIF(torch.autograd.Function):
    """spikes = FusedAffineLIF.apply(x, scale, shift, params[, residual]) for x [T, B, C, *spatial]:
    the per-channel affine (e.g. BatchNorm's gamma/sigma, beta - mu gamma/sigma) and, when
    given, the residual shortcut (same shape as x) are folded into the LIF prologue
    (SURVEY 8(f) f4), so neither the normalised tensor nor the sum touches HBM."""

    @staticmethod
    def forward(ctx, x, scale, shift, params: LIFParams, residual=None):
        T, B, C = x.shape[:3]
        HW = x[0, 0, 0].numel()
        x2 = x.reshape(T, -1)
        x2 = x2 if x2.is_contiguous() else x2.contiguous()
        r2 = None
        if residual is not None:   # the spiking-ResNet shortcut added to the LIF input
            r2 = residual.reshape(T, -1).to(x.dtype)
            r2 = r2 if r2.is_contiguous() else r2.contiguous()
        spec = AffineSpec(scale.contiguous(), shift.contiguous(), C, HW)
        fwd = lif_forward_affine(x2, params, spec, spike_fmt="io", return_v_final=False, residual=r2)
        ctx.save_for_backward(x2, fwd.saved, spec.scale, spec.shift, fwd.residual)
        ctx.params, ctx.cshape, ctx.C, ctx.HW = params, fwd.shape, C, HW
        ctx.shape = x.shape
        ctx.res_shape = None if residual is None else (residual.shape, residual.dtype)
        return fwd.spikes.reshape(x.shape)

    @staticmethod
    def backward(ctx, grad_spikes):
        x2, saved, scale, shift, r2 = ctx.saved_tensors
        fwd = LIFForward(None, saved, None, x2, None, ctx.params, ctx.cshape)
        fwd.affine = AffineSpec(scale, shift, ctx.C, ctx.HW)
        fwd.residual = r2
        T = grad_spikes.shape[0]
        out = lif_backward_affine(grad_spikes.reshape(T, -1).to(x2.dtype), fwd, return_grad_v_init=False)
        gres = None
        if ctx.res_shape is not None:
            shape, dtype = ctx.res_shape
            gres = out[4].reshape(shape).to(dtype)
        return out[0].reshape(ctx.shape), out[2], out[3], None, gres


class AffineLIFLayer(torch.nn.Module):
    """Per-channel affine (learnable scale / shift, init 1 / 0) fused with a LIF layer.
    Input [T, B, C, *spatial] (time-major)."""

    def __init__(self, channels: int, params: Optional[LIFParams] = None, **kw):
        super().__init__()
        self.params = params if params is not None else LIFParams(**kw)
        self.scale = torch.nn.Parameter(torch.ones(channels))
        self.shift = torch.nn.Parameter(torch.zeros(channels))

    def forward(self, x, residual=None):
        """spikes = LIF(scale[c] x + shift[c] (+ residual)); residual has x's shape."""
        return FusedAffineLIF.apply(x, self.scale, self.shift, self.params, residual)
