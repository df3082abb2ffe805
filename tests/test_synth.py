"""The seeded input generator (snn_synth): deterministic, shard-consistent, N(0,1)-shaped."""
import torch

import snn_synth


def test_moments_and_support():
    x = snn_synth.normal_tensor(1234, 32, 8192)
    assert abs(x.mean().item()) < 0.01 and abs(x.std().item() - 1.0) < 0.01
    assert x.abs().max().item() <= 6.0


def test_shard_segment_and_column_views_are_bitwise_consistent():
    whole = snn_synth.normal_tensor(7, 40, 3000, mean=1.0)
    part = snn_synth.normal_tensor(7, 11, 500, n_global=3000, n_offset=1234, t_offset=20, mean=1.0)
    assert torch.equal(part, whole[20:31, 1234:1734])
    cols = [0, 1, 2999, 1500]
    assert torch.equal(snn_synth.normal_columns(7, 40, 3000, cols, mean=1.0), whole[:, cols])


def test_seeds_differ_and_bf16_is_rounded_fp32():
    a = snn_synth.normal_tensor(1, 4, 64)
    b = snn_synth.normal_tensor(2, 4, 64)
    assert not torch.equal(a, b)
    c = snn_synth.normal_tensor(1, 4, 64, dtype=torch.bfloat16)
    assert torch.equal(c, a.to(torch.bfloat16))
