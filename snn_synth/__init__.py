"""Seeded, counter-based synthetic inputs shared by tests, bench.py and smoke().

Holds NONE of the method's arithmetic: it only turns (seed, flat index) into numbers.
Both the oracle side (host, any subset of indices) and the GPU side (whole tensors on
the device) call the same torch integer/float code, so a sampled column regenerated on
the host is bit-identical to the same column generated on the device -- no oracle input
is ever copied back from the CUDA path.

Generator: element i of stream ``seed`` draws four splitmix64 words
h_j = splitmix64(seed_key + 4 i + j), j = 0..3, splits each into three 20-bit fields, and
returns the Irwin-Hall(12) variate  z = sum_{m<12} u_m 2^-20 - 6  (mean 0, variance 1,
support [-6, 6]; every step is exact in fp32 because sum u_m < 12 * 2^20 < 2^24), then
``mean + std * z`` (two correctly-rounded fp32 ops, identical on CPU and GPU).
DESIGN.md "Input recipe" states the distributions each workload uses.
"""
from __future__ import annotations

import torch

_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    """uint64 constant -> the int64 with the same bits."""
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


_GAMMA = _s64(0x9E3779B97F4A7C15)
_MUL1 = _s64(0xBF58476D1CE4E5B9)
_MUL2 = _s64(0x94D049BB133111EB)


def _shr(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser of (x + gamma) on int64 tensors (wrapping arithmetic)."""
    z = x + _GAMMA
    z = (z ^ _shr(z, 30)) * _MUL1
    z = (z ^ _shr(z, 27)) * _MUL2
    return z ^ _shr(z, 31)


def seed_key(seed: int) -> int:
    return int(splitmix64(torch.tensor([_s64(seed)], dtype=torch.int64)).item())


def normal_at(seed: int, idx: torch.Tensor, mean: float = 0.0, std: float = 1.0) -> torch.Tensor:
    """Approximately-normal fp32 variates for flat indices ``idx`` (int64, any device)."""
    key = seed_key(seed)
    base = idx.to(torch.int64) * 4 + key
    acc = torch.zeros(idx.shape, dtype=torch.int64, device=idx.device)
    for j in range(4):
        h = splitmix64(base + j)
        mask = (1 << 20) - 1
        acc += (h & mask) + (_shr(h, 20) & mask) + (_shr(h, 40) & mask)
    z = acc.to(torch.float32) * (2.0 ** -20) - 6.0
    if std != 1.0:
        z = z * std
    if mean != 0.0:
        z = z + mean
    return z


def normal_tensor(seed: int, T: int, N: int, *, n_global: int | None = None, n_offset: int = 0,
                  t_offset: int = 0, mean: float = 0.0, std: float = 1.0,
                  device="cpu", dtype=torch.float32, rows_per_chunk: int = 64) -> torch.Tensor:
    """[T, N] block of the global [T_global, n_global] stream at (t_offset, n_offset).

    Element (t, n) is ``normal_at(seed, (t + t_offset) * n_global + n + n_offset)``, so a
    neuron shard, a time segment or a sampled column set regenerates exactly the bits a
    whole-tensor run sees.  Generated in row chunks to bound temporaries."""
    n_global = N if n_global is None else n_global
    out = torch.empty((T, N), dtype=dtype, device=device)
    cols = torch.arange(N, dtype=torch.int64, device=device) + n_offset
    for t0 in range(0, T, rows_per_chunk):
        t1 = min(T, t0 + rows_per_chunk)
        rows = torch.arange(t0, t1, dtype=torch.int64, device=device) + t_offset
        idx = rows[:, None] * n_global + cols[None, :]
        out[t0:t1] = normal_at(seed, idx, mean, std).to(dtype)
    return out


def normal_columns(seed: int, T: int, n_global: int, cols, *, t_offset: int = 0,
                   mean: float = 0.0, std: float = 1.0, dtype=torch.float32) -> torch.Tensor:
    """Host-side [T, len(cols)] gather of the global stream (for sampled-column parity)."""
    cols = torch.as_tensor(cols, dtype=torch.int64)
    rows = torch.arange(T, dtype=torch.int64) + t_offset
    idx = rows[:, None] * n_global + cols[None, :]
    return normal_at(seed, idx, mean, std).to(dtype)
