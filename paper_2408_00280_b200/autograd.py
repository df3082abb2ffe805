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

from .lif import LIFParams, lif_backward, lif_forward


class FusedLIF(torch.autograd.Function):
    """spikes = FusedLIF.apply(x, params, v_init, save_mode); x: CUDA [T, N] fp32/bf16.
    Spikes are returned in x's dtype (0/1), the form the next ANN operator consumes."""

    @staticmethod
    def forward(ctx, x: torch.Tensor, params: LIFParams, v_init: Optional[torch.Tensor] = None,
                save_mode: str = "recompute"):
        x = x if x.stride(-1) == 1 else x.contiguous()
        fwd = lif_forward(x, params, v_init=v_init, spike_fmt="io", save_mode=save_mode,
                          return_v_final=False)
        ctx.fwd = fwd
        ctx.has_v_init = v_init is not None
        return fwd.spikes

    @staticmethod
    def backward(ctx, grad_spikes: torch.Tensor):
        fwd = ctx.fwd
        gx, gvi = lif_backward(grad_spikes.to(fwd.x.dtype), fwd,
                               return_grad_v_init=ctx.has_v_init and ctx.needs_input_grad[2])
        ctx.fwd = None
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
