"""Comparison helpers for two GPU decompositions of the same attention (test infrastructure)."""
import torch


def assert_bf16_close(a: torch.Tensor, b: torch.Tensor, ulps: float = 2.0, atol: float = 4e-3):
    """|a - b| <= ulps * bf16-ulp(max(|a|, |b|)) + atol: two roundings of the same fp32 sum to
    bf16 may land one ulp apart (2^-7 relative at the top of each binade)."""
    a = a.float()
    b = b.float()
    mag = torch.maximum(a.abs(), b.abs())
    ulp = torch.exp2(torch.floor(torch.log2(mag.clamp_min(1e-30))) - 7)
    bad = (a - b).abs() > ulps * ulp + atol
    assert not bool(bad.any()), f"max diff {(a - b).abs().max().item():.3e}"
