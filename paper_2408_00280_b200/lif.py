"""Functional torch-facing API over the C ABI (marshalling only; every step of the LIF
path runs in the CUDA kernels of libsnn_lif.so).

    lif_forward(x, params, ...)   -> LIFForward(spikes, saved, v_final, ...)
    lif_backward(grad_spikes, fwd, ...) -> (grad_x, grad_v_init)

``x`` is a CUDA tensor [T, N] (fp32 or bf16) whose rows may be strided (``x.stride(1)``
must be 1; ``ld = x.stride(0)``), so a neuron-shard column view of a wider tensor is
passed without a copy.  Kernels are enqueued on ``torch.cuda.current_stream()``.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional

import torch

from . import _lib

_SPIKE_FMTS = {"u8": _lib.SNN_SPK_U8, "bits": _lib.SNN_SPK_BITS, "io": _lib.SNN_SPK_IO}
_SAVE_MODES = {"h": _lib.SNN_SAVE_H, "recompute": _lib.SNN_SAVE_RECOMPUTE, "none": _lib.SNN_SAVE_NONE}
_DTYPES = {torch.float32: _lib.SNN_F32, torch.bfloat16: _lib.SNN_BF16}


@dataclass(frozen=True)
class LIFParams:
    """LIF hyper-parameters (include/snn_lif.h ``snn_lif_params``).

    Defaults are the paper's: k_tau = 0.2 (tau = 1.25), V_th = 0.3,
    V_rest = 0, hard reset, input not decayed (Eq. 1), gradient through the reset (Eq. 3),
    sigmoid surrogate with alpha = 4."""
    tau: float = 1.25
    v_th: float = 0.3
    v_reset: float = 0.0
    reset: str = "hard"          # "hard" | "soft"
    decay_input: bool = False    # True: H = V + (X - (V - V_reset))/tau (north star)
    detach_reset: bool = False
    surrogate: str = "sigmoid"   # "sigmoid" | "atan"
    alpha: float = 4.0

    @staticmethod
    def paper() -> "LIFParams":
        return LIFParams()

    @staticmethod
    def north_star(**kw) -> "LIFParams":
        """BASELINE.json configs[0]: tau=2, V_th=1, V_reset=0, hard, sigmoid, decay_input."""
        return replace(LIFParams(tau=2.0, v_th=1.0, v_reset=0.0, decay_input=True), **kw)

    def to_c(self) -> _lib.snn_lif_params:
        """The C struct, built once per (frozen) parameter set and reused by every call."""
        c = self.__dict__.get("_c_struct")
        if c is None:
            c = self._build_c()
            object.__setattr__(self, "_c_struct", c)
        return c

    def _build_c(self) -> _lib.snn_lif_params:
        return _lib.snn_lif_params(
            float(self.tau), float(self.v_th), float(self.v_reset),
            {"hard": _lib.SNN_RESET_HARD, "soft": _lib.SNN_RESET_SOFT}[self.reset],
            int(bool(self.decay_input)), int(bool(self.detach_reset)),
            {"sigmoid": _lib.SNN_SURR_SIGMOID, "atan": _lib.SNN_SURR_ATAN}[self.surrogate],
            float(self.alpha))


@dataclass
class LIFForward:
    """Result of lif_forward: spikes plus what the backward needs."""
    spikes: torch.Tensor
    saved: Optional[torch.Tensor]
    v_final: Optional[torch.Tensor]
    x: torch.Tensor
    v_init: Optional[torch.Tensor]
    params: LIFParams
    shape: _lib.snn_lif_shape


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _stream(device: Optional[torch.device] = None) -> int:
    """cudaStream_t of torch's current stream on `device` (default: the current device)."""
    idx = torch.cuda.current_device() if device is None or device.index is None else device.index
    return torch._C._cuda_getCurrentRawStream(idx)


def _check_2d(name: str, t: torch.Tensor) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if t.dim() != 2 or (t.size(1) > 1 and t.stride(1) != 1):
        raise ValueError(f"{name} must be [T, N] with unit column stride, got {tuple(t.shape)} "
                         f"strides {t.stride()}")


def _vec(name, t, N, device):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == torch.float32 and t.numel() == N and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous fp32 CUDA tensor of {N} elements")
    return t


_SHAPES: dict = {}      # (T, N, ld, dtype, spike_fmt, save_mode) -> (snn_lif_shape, saved bytes)


def _shape_entry(x: torch.Tensor, spike_fmt: str, save_mode: str):
    """The C shape struct and its saved-buffer size, built once per distinct layout (host
    overhead of an eager call; the structs are only read by the library)."""
    T, N = x.shape
    ld = max(x.stride(0) if T > 1 else N, N)
    key = (T, N, ld, x.dtype, spike_fmt, save_mode)
    e = _SHAPES.get(key)
    if e is None:
        shape = _lib.snn_lif_shape(T, N, ld, _DTYPES[x.dtype], _SPIKE_FMTS[spike_fmt], _SAVE_MODES[save_mode])
        # the saved size depends on the shape only (any valid params give the same answer)
        e = (shape, _lib.snn_lif_saved_bytes(LIFParams().to_c(), shape))
        if len(_SHAPES) > 4096:
            _SHAPES.clear()
        _SHAPES[key] = e
    return e


def make_shape(x: torch.Tensor, spike_fmt: str, save_mode: str) -> _lib.snn_lif_shape:
    return _shape_entry(x, spike_fmt, save_mode)[0]


def saved_bytes(params: LIFParams, shape: _lib.snn_lif_shape) -> int:
    return _lib.snn_lif_saved_bytes(params.to_c(), shape)


def alloc_spikes(x: torch.Tensor, spike_fmt: str, ld: Optional[int] = None) -> torch.Tensor:
    """Spike output for x [T, N]: u8 / io rows of stride ``ld`` (default N; the kernels walk
    every [T, N] operand with x's row stride), bits as dense [T, ceil(N/32)] words."""
    T, N = x.shape
    if ld is not None and ld != N and spike_fmt != "bits":
        dt = torch.uint8 if spike_fmt == "u8" else x.dtype
        return torch.empty((T, ld), dtype=dt, device=x.device)[:, :N]
    if spike_fmt == "u8":
        return torch.empty((T, N), dtype=torch.uint8, device=x.device)
    if spike_fmt == "bits":
        return torch.empty((T, (N + 31) // 32), dtype=torch.int32, device=x.device)
    return torch.empty((T, N), dtype=x.dtype, device=x.device)


def lif_forward(x: torch.Tensor, params: LIFParams = LIFParams(), *,
                v_init: Optional[torch.Tensor] = None, spike_fmt: str = "u8",
                save_mode: str = "recompute", return_v_final: bool = True,
                spikes: Optional[torch.Tensor] = None, saved: Optional[torch.Tensor] = None,
                v_final: Optional[torch.Tensor] = None) -> LIFForward:
    """Eq. 1-2 over all T steps in one kernel launch (fusedForwardLIF).

    spike_fmt: "u8" ([T, N] uint8), "bits" ([T, ceil(N/32)] int32 words, bit j of word w =
    neuron 32w+j) or "io" (x's dtype, 0/1).  save_mode: "recompute" (V checkpoints every
    16 steps), "h" (fp32 H every step) or "none" (inference).  Preallocated outputs may
    be passed (spikes must then have row stride ld for u8/io)."""
    _check_2d("x", x)
    if x.dtype not in _DTYPES:
        raise ValueError(f"x dtype {x.dtype} unsupported (fp32 / bf16)")
    T, N = x.shape
    shape, nbytes = _shape_entry(x, spike_fmt, save_mode)
    cp = params.to_c()
    v_init = _vec("v_init", v_init, N, x.device)
    if spikes is None:   # keep the caller's ld for views: [T, ld] with its first N columns used
        spikes = alloc_spikes(x, spike_fmt, shape.ld)
    if save_mode != "none" and saved is None:
        saved = torch.empty(nbytes // 4, dtype=torch.float32, device=x.device)
    if return_v_final and v_final is None:
        v_final = torch.empty(N, dtype=torch.float32, device=x.device)
    _lib.snn_lif_forward(cp, shape, _ptr(x), _ptr(v_init), _ptr(spikes),
                         _ptr(saved) if save_mode != "none" else None, _ptr(v_final), _stream(x.device))
    return LIFForward(spikes, saved if save_mode != "none" else None, v_final, x, v_init,
                      params, shape)


def lif_backward(grad_spikes: torch.Tensor, fwd: LIFForward, *,
                 grad_v_final: Optional[torch.Tensor] = None, return_grad_v_init: bool = True,
                 grad_x: Optional[torch.Tensor] = None):
    """Eq. 3 over t = T-1..0 in one kernel launch (fusedBackwardLIF).
    Returns (grad_x [T, N] in x's dtype, grad_v_init [N] fp32 or None)."""
    if not grad_spikes.is_cuda:
        raise ValueError("grad_spikes must be a CUDA tensor (no CPU path exists)")
    if grad_spikes.dim() == 2 and grad_spikes.size(1) > 1 and grad_spikes.stride(1) != 1:
        grad_spikes = grad_spikes.contiguous()   # e.g. the expanded ones of y.sum().backward()
    _check_2d("grad_spikes", grad_spikes)
    x = fwd.x
    T, N = x.shape
    if tuple(grad_spikes.shape) != (T, N) or grad_spikes.dtype != x.dtype:
        raise ValueError("grad_spikes must match x in shape and dtype")
    if fwd.saved is None:
        raise ValueError("forward ran with save_mode='none'; nothing to differentiate")
    ld = fwd.shape.ld
    if T > 1 and grad_spikes.stride(0) != ld:
        grad_spikes = grad_spikes.contiguous() if ld == N else _restride(grad_spikes, ld)
    if grad_x is None:
        grad_x = torch.empty((T, ld), dtype=x.dtype, device=x.device)[:, :N]
    grad_v_final = _vec("grad_v_final", grad_v_final, N, x.device)
    grad_v_init = torch.empty(N, dtype=torch.float32, device=x.device) if return_grad_v_init else None
    _lib.snn_lif_backward(fwd.params.to_c(), fwd.shape, _ptr(grad_spikes), _ptr(x),
                          _ptr(fwd.v_init), _ptr(fwd.saved), _ptr(grad_v_final), _ptr(grad_x),
                          _ptr(grad_v_init), _stream(x.device))
    return grad_x, grad_v_init


def _restride(t: torch.Tensor, ld: int) -> torch.Tensor:
    T, N = t.shape
    out = torch.empty((T, ld), dtype=t.dtype, device=t.device)[:, :N]
    out.copy_(t)
    return out


def unpack_bits(words: torch.Tensor, N: int) -> torch.Tensor:
    """[T, ceil(N/32)] int32 spike words -> [T, N] uint8 (a view helper for tests/users)."""
    T, W = words.shape
    shifts = torch.arange(32, device=words.device, dtype=torch.int32)
    bits = (words.unsqueeze(-1) >> shifts) & 1
    return bits.reshape(T, W * 32)[:, :N].to(torch.uint8)


# ----------------------------------------------------------------------------- baseline

def lif_serial(x: torch.Tensor, grad_spikes: torch.Tensor, params: LIFParams = LIFParams(), *,
               v_init: Optional[torch.Tensor] = None):
    """The paper's "Serial (CUDA)" baseline (Fig. 3): T forward launches then T backward
    launches, state through HBM between steps.  Comparison only; bitwise equal to the fused
    path.  x, grad_spikes: contiguous CUDA [T, N].  Returns (spikes u8, H, v_final, grad_x,
    grad_v_init)."""
    T, N = x.shape
    x = x.contiguous(); grad_spikes = grad_spikes.contiguous()
    cp, io, st = params.to_c(), _DTYPES[x.dtype], _stream()
    v = (v_init.clone() if v_init is not None else
         torch.full((N,), float(params.v_reset), dtype=torch.float32, device=x.device))
    S = torch.empty((T, N), dtype=torch.uint8, device=x.device)
    H = torch.empty((T, N), dtype=torch.float32, device=x.device)
    for t in range(T):
        _lib.snn_lif_serial_forward_step(cp, io, N, _ptr(x[t]), _ptr(v), _ptr(S[t]), _ptr(H[t]), st)
    gv = torch.zeros(N, dtype=torch.float32, device=x.device)
    gX = torch.empty_like(x)
    for t in range(T - 1, -1, -1):
        _lib.snn_lif_serial_backward_step(cp, io, N, _ptr(grad_spikes[t]), _ptr(H[t]), _ptr(gv),
                                          _ptr(gX[t]), st)
    return S, H, v, gX, gv



# ----------------------------------------------------------------------------- f4: affine prologue

@dataclass
class AffineSpec:
    """Per-channel affine folded into the LIF input: X' = scale[c] X + shift[c],
    c = (n / HW) % C (include/snn_lif.h snn_lif_affine)."""
    scale: torch.Tensor   # [C] fp32 CUDA
    shift: torch.Tensor   # [C] fp32 CUDA
    C: int
    HW: int

    def to_c(self, residual: Optional[torch.Tensor] = None,
             grad_residual: Optional[torch.Tensor] = None) -> _lib.snn_lif_affine:
        for name, t in (("scale", self.scale), ("shift", self.shift)):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.numel() == self.C):
                raise ValueError(f"affine {name} must be a contiguous fp32 CUDA tensor of C={self.C}")
        return _lib.snn_lif_affine(self.scale.data_ptr(), self.shift.data_ptr(), self.C, self.HW,
                                   _ptr(residual), _ptr(grad_residual))


def _like_x(name: str, t: torch.Tensor, x: torch.Tensor, ld: int) -> torch.Tensor:
    """A [T, N] operand laid out like x (same dtype, device, row stride ld)."""
    if t.shape != x.shape or t.dtype != x.dtype or t.device != x.device:
        raise ValueError(f"{name} must match x: {tuple(x.shape)} {x.dtype} on {x.device}")
    if t.dim() == 2 and t.size(1) > 1 and t.stride(1) != 1:
        t = t.contiguous()
    if t.shape[0] > 1 and t.stride(0) != ld:
        t = t.contiguous() if ld == t.shape[1] else _restride(t, ld)
    return t


def lif_forward_affine(x: torch.Tensor, params: LIFParams, affine: AffineSpec, *,
                       v_init: Optional[torch.Tensor] = None, spike_fmt: str = "u8",
                       return_v_final: bool = True,
                       residual: Optional[torch.Tensor] = None) -> LIFForward:
    """Forward with the affine prologue fused in (RECOMPUTE save mode: the backward re-reads x).
    ``residual`` [T, N] (x's dtype): the LIF input becomes scale[c] x + shift[c] + residual
    (the spiking-ResNet shortcut); the backward then also returns dL/dresidual."""
    _check_2d("x", x)
    T, N = x.shape
    shape = make_shape(x, spike_fmt, "recompute")
    if residual is not None:
        residual = _like_x("residual", residual, x, shape.ld)
    cp = params.to_c()
    v_init = _vec("v_init", v_init, N, x.device)
    spikes = alloc_spikes(x, spike_fmt, shape.ld)
    saved = torch.empty(_lib.snn_lif_saved_bytes(cp, shape) // 4, dtype=torch.float32, device=x.device)
    v_final = torch.empty(N, dtype=torch.float32, device=x.device) if return_v_final else None
    ca = affine.to_c(residual)
    _lib.snn_lif_forward_affine(cp, shape, _ptr(x), _ptr(v_init), ca, _ptr(spikes), _ptr(saved),
                                _ptr(v_final), _stream())
    f = LIFForward(spikes, saved, v_final, x, v_init, params, shape)
    f.affine = affine
    f.residual = residual
    return f


def lif_backward_affine(grad_spikes: torch.Tensor, fwd: LIFForward, *,
                        grad_v_final: Optional[torch.Tensor] = None, return_grad_v_init: bool = True):
    """Returns (grad_x [T, N] w.r.t. the raw input, grad_v_init, grad_scale [C], grad_shift [C]),
    plus grad_residual [T, N] as a fifth element when the forward had a residual."""
    x = fwd.x
    T, N = x.shape
    if grad_spikes.dim() == 2 and grad_spikes.size(1) > 1 and grad_spikes.stride(1) != 1:
        grad_spikes = grad_spikes.contiguous()
    _check_2d("grad_spikes", grad_spikes)
    ld = fwd.shape.ld
    if T > 1 and grad_spikes.stride(0) != ld:
        grad_spikes = grad_spikes.contiguous() if ld == N else _restride(grad_spikes, ld)
    af = fwd.affine
    grad_x = torch.empty((T, ld), dtype=x.dtype, device=x.device)[:, :N]
    gvi = torch.empty(N, dtype=torch.float32, device=x.device) if return_grad_v_init else None
    npad = (N + 3) // 4 * 4                      # each partial row 16-byte aligned
    part = torch.empty((2, npad), dtype=torch.float32, device=x.device)
    gsc = torch.empty(af.C, dtype=torch.float32, device=x.device)
    gsh = torch.empty(af.C, dtype=torch.float32, device=x.device)
    res = getattr(fwd, "residual", None)
    grad_res = None if res is None else torch.empty((T, ld), dtype=x.dtype, device=x.device)[:, :N]
    _lib.snn_lif_backward_affine(fwd.params.to_c(), fwd.shape, _ptr(grad_spikes), _ptr(x), _ptr(fwd.v_init),
                                 _ptr(fwd.saved),
                                 _ptr(_vec("grad_v_final", grad_v_final, N, x.device)),
                                 af.to_c(res, grad_res), _ptr(grad_x), _ptr(gvi), _ptr(part[0]),
                                 _ptr(part[1]), _ptr(gsc), _ptr(gsh), _stream())
    if res is not None:
        return grad_x, gvi, gsc, gsh, grad_res
    return grad_x, gvi, gsc, gsh


def host_workspace(T: int, N: int, params: LIFParams, dtype=torch.float32, *, spike_fmt: str = "u8",
                   save_mode: str = "recompute", chunk_neurons: int = 0, nslots: int = 3,
                   device=None) -> torch.Tensor:
    """Device staging memory for lif_fwd_bwd_host (allocate once, reuse across calls)."""
    shape = _lib.snn_lif_shape(T, N, N, _DTYPES[dtype], _SPIKE_FMTS[spike_fmt], _SAVE_MODES[save_mode])
    nbytes = _lib.snn_lif_host_workspace_bytes(params.to_c(), shape, chunk_neurons, nslots)
    if nbytes == 0:
        raise ValueError("invalid shape / chunk_neurons / nslots for the host-buffer path")
    return torch.empty(nbytes, dtype=torch.uint8, device=device or torch.device("cuda"))


def lif_fwd_bwd_host(x: torch.Tensor, grad_spikes: torch.Tensor, params: LIFParams = LIFParams(), *,
                     spike_fmt: str = "u8", save_mode: str = "recompute",
                     spikes: Optional[torch.Tensor] = None, grad_x: Optional[torch.Tensor] = None,
                     chunk_neurons: int = 0, nslots: int = 3,
                     workspace: Optional[torch.Tensor] = None):
    """One layer's forward + backward on HOST tensors (pin them for full PCIe speed):
    x, grad_spikes [T, N] fp32/bf16 CPU -> (spikes, grad_x) CPU.  Streams neuron chunks
    through the device with copy-in, the fused kernels and copy-out overlapped
    (snn_lif_fwd_bwd_host); blocks until the outputs are in host memory."""
    for name, t in (("x", x), ("grad_spikes", grad_spikes)):
        if t.is_cuda or t.dim() != 2 or (t.size(1) > 1 and t.stride(1) != 1):
            raise ValueError(f"{name} must be a [T, N] host tensor with unit column stride")
    if grad_spikes.shape != x.shape or grad_spikes.dtype != x.dtype or grad_spikes.stride() != x.stride():
        raise ValueError("grad_spikes must match x in shape, dtype and strides")
    T, N = x.shape
    shape = make_shape(x, spike_fmt, save_mode)
    if spikes is None:
        pin = x.is_pinned()
        if spike_fmt == "u8":
            spikes = torch.empty((T, shape.ld), dtype=torch.uint8, pin_memory=pin)[:, :N]
        elif spike_fmt == "bits":
            spikes = torch.empty((T, (N + 31) // 32), dtype=torch.int32, pin_memory=pin)
        else:
            spikes = torch.empty((T, shape.ld), dtype=x.dtype, pin_memory=pin)[:, :N]
    if grad_x is None:
        grad_x = torch.empty((T, shape.ld), dtype=x.dtype, pin_memory=x.is_pinned())[:, :N]
    if grad_x.stride() != x.stride() or grad_x.dtype != x.dtype:
        raise ValueError("grad_x must match x in dtype and strides")
    cp = params.to_c()
    need = _lib.snn_lif_host_workspace_bytes(cp, shape, chunk_neurons, nslots)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device="cuda")
    _lib.snn_lif_fwd_bwd_host(cp, shape, x.data_ptr(), grad_spikes.data_ptr(), spikes.data_ptr(),
                              grad_x.data_ptr(), chunk_neurons, nslots, workspace.data_ptr(),
                              workspace.numel(), _stream())
    return spikes, grad_x


# ----------------------------------------------------------------------------- plans

class LIFPlan:
    """A fused LIF layer bound to fixed buffers: the C ABI validates the call once
    (snn_lif_plan_create: parameters, layout, kernel variant, TMA tensor maps) and every
    ``forward()`` / ``backward()`` replays only the kernel launches on torch's current
    stream -- for serving loops or training steps that reuse their activation buffers.
    Write new inputs into ``x`` / ``grad_spikes`` in place between calls; results land in
    ``spikes`` / ``grad_x`` (bitwise what lif_forward / lif_backward return)."""

    def __init__(self, x: torch.Tensor, params: LIFParams = LIFParams(), *, spike_fmt: str = "u8",
                 save_mode: str = "recompute", v_init: Optional[torch.Tensor] = None,
                 grad_spikes: Optional[torch.Tensor] = None, grad_v_final: Optional[torch.Tensor] = None,
                 with_v_final: bool = False, with_grad_v_init: bool = False,
                 affine: Optional["AffineSpec"] = None, residual: Optional[torch.Tensor] = None):
        """affine / residual: the f4 prologue (lif_forward_affine); the backward then also fills
        ``grad_scale`` / ``grad_shift`` (and ``grad_residual``).  save_mode must be "recompute"
        (or "none" for a forward-only, BN-folded inference plan)."""
        _check_2d("x", x)
        T, N = x.shape
        self.x, self.params, self.device = x, params, x.device
        self.shape, nbytes = _shape_entry(x, spike_fmt, save_mode)
        self.v_init = _vec("v_init", v_init, N, x.device)
        self.spikes = alloc_spikes(x, spike_fmt, self.shape.ld)
        self.saved = torch.empty(nbytes // 4, dtype=torch.float32, device=x.device) if save_mode != "none" else None
        self.v_final = torch.empty(N, dtype=torch.float32, device=x.device) if with_v_final else None
        self.grad_spikes = grad_spikes
        self.grad_x = self.grad_v_init = None
        if grad_spikes is not None:
            _check_2d("grad_spikes", grad_spikes)
            if tuple(grad_spikes.shape) != (T, N) or grad_spikes.dtype != x.dtype or \
                    (T > 1 and grad_spikes.stride(0) != self.shape.ld):
                raise ValueError("grad_spikes must match x in shape, dtype and row stride")
            self.grad_x = torch.empty((T, self.shape.ld), dtype=x.dtype, device=x.device)[:, :N]
            self.grad_v_init = torch.empty(N, dtype=torch.float32, device=x.device) if with_grad_v_init else None
        self.grad_v_final = _vec("grad_v_final", grad_v_final, N, x.device)
        if affine is None:
            if residual is not None:
                raise ValueError("residual needs an affine (use scale 1, shift 0 for a plain shortcut)")
            self._plan = _lib.snn_lif_plan_create(
                params.to_c(), self.shape, _ptr(x), _ptr(self.v_init), _ptr(self.spikes), _ptr(self.saved),
                _ptr(self.v_final), _ptr(grad_spikes), _ptr(self.grad_v_final), _ptr(self.grad_x),
                _ptr(self.grad_v_init))
            return
        self.affine, self.residual = affine, residual
        if residual is not None:
            residual = self.residual = _like_x("residual", residual, x, self.shape.ld)
        self.grad_residual = self.grad_scale = self.grad_shift = self._part = None
        if grad_spikes is not None:
            if residual is not None:
                self.grad_residual = torch.empty((T, self.shape.ld), dtype=x.dtype, device=x.device)[:, :N]
            self._part = torch.empty((2, (N + 3) // 4 * 4), dtype=torch.float32, device=x.device)
            self.grad_scale = torch.empty(affine.C, dtype=torch.float32, device=x.device)
            self.grad_shift = torch.empty(affine.C, dtype=torch.float32, device=x.device)
        self._c_affine = affine.to_c(residual, self.grad_residual)   # kept alive with the plan
        self._plan = _lib.snn_lif_plan_create_affine(
            params.to_c(), self.shape, _ptr(x), _ptr(self.v_init), self._c_affine, _ptr(self.spikes),
            _ptr(self.saved), _ptr(self.v_final), _ptr(grad_spikes), _ptr(self.grad_v_final), _ptr(self.grad_x),
            _ptr(self.grad_v_init), None if self._part is None else _ptr(self._part[0]),
            None if self._part is None else _ptr(self._part[1]), _ptr(self.grad_scale), _ptr(self.grad_shift))

    def forward(self) -> torch.Tensor:
        _lib.snn_lif_plan_forward(self._plan, _stream(self.device))
        return self.spikes

    def backward(self) -> torch.Tensor:
        _lib.snn_lif_plan_backward(self._plan, _stream(self.device))
        return self.grad_x

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan:
            _lib.snn_lif_plan_destroy(plan)
            self._plan = None
