"""tcgen05 building blocks of the extend kernel (descriptors, TMEM layouts) vs torch."""
import pytest
import torch

from paper_2511_20048_b200 import spa

pytestmark = pytest.mark.gpu


def test_umma_selftest_matches_torch():
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((128, 128), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((32, 128), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((32, 128), generator=g, device="cuda").to(torch.bfloat16)
    s, o = spa.umma_selftest(q, k, v)
    torch.cuda.synchronize()
    s_ref = q.double() @ k.double().T
    assert (s.double() - s_ref).abs().max().item() < 1e-3
    o_ref = s.to(torch.bfloat16).double() @ v.double()
    assert (o.double() - o_ref).abs().max().item() < 1e-2 * o_ref.abs().max().item()
