"""Caller-owned plan workspace (include/spa.h spa_plan_set_workspace; SURVEY.md Sec. 8(b):
all device memory is caller-owned): a torch-allocated workspace, SPA_ERR_WORKSPACE when it
is too small, and plan + decode captured in one CUDA graph whose replays match the oracle."""
import numpy as np
import pytest
import torch

from harness import LSE_TOL, O_TOL, GpuBatch, bits_to_torch, compare
from oracle.replay import Replay
from paper_2511_20048_b200 import spa
from spa_inputs import families, workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu(cuda_device):
    spa.lib()
    yield


def _batch(seed=5):
    rec = workloads.sweep(12, 0.75, seed=seed)   # parents with 3 forks (20 rows per group)
    rec.groups = rec.groups[:3]
    for g in rec.groups:
        g.prefix = 300 + g.prefix % 200
    inp = families.make_inputs(rec, "needle_shared_pos")
    return inp, GpuBatch(inp)


def test_fixed_workspace_too_small_then_grown():
    inp, gb = _batch()
    small = torch.empty(1024, dtype=torch.uint8, device="cuda")
    plan = spa.Plan(gb.pool, split_pages=3, workspace=small)
    st = plan.plan(gb.reqs, check=False)
    assert st == spa.SPA_ERR_WORKSPACE
    need = plan.workspace_size()
    assert need > 1024
    m = inp.recipe.model
    q = bits_to_torch(inp.q[0]).contiguous()
    o = torch.empty((len(gb.reqs), m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((len(gb.reqs), m.num_q_heads), dtype=torch.float32, device="cuda")
    st = spa.lib().spa_decode_attention(plan.h, 0, spa._ptr(q), q.stride(0), q.stride(1), spa._ptr(o), o.stride(0),
                                        o.stride(1), spa._ptr(lse), lse.stride(0), lse.stride(1), 1.0, None)
    assert st == spa.SPA_ERR_WORKSPACE                         # refused: the plan never reached the device
    plan.set_workspace(torch.empty(need, dtype=torch.uint8, device="cuda"))   # exactly the need
    plan.plan(gb.reqs)
    assert plan.stats()["n_records"] > 0                       # split partials live in the workspace too
    rp = Replay(inp)
    o, lse = gb.decode(plan, 0)
    eo, el = compare(o, lse, *rp.expected(0, inp.q[0]))
    assert eo <= O_TOL and el <= LSE_TOL, (eo, el)


def test_plan_and_decode_captured_in_a_cuda_graph():
    inp, gb = _batch(9)
    m = inp.recipe.model
    L = len(inp.layers)
    plan = spa.Plan(gb.pool, split_pages=3)
    plan.plan(gb.reqs)                       # sizes the pinned staging buffer and the workspace
    ws = torch.empty(plan.workspace_size() + 4096, dtype=torch.uint8, device="cuda")
    plan.set_workspace(ws)
    N = len(gb.reqs)
    q = torch.stack([bits_to_torch(inp.q[li]) for li in range(L)]).contiguous()
    o = torch.zeros((L, N, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device="cuda")
    lse = torch.zeros((L, N, m.num_q_heads), dtype=torch.float32, device="cuda")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.plan(gb.reqs, stream=s)         # one warm call on the capture stream
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            plan.plan(gb.reqs, stream=s)     # the upload is a memcpy node (re-zeroes the counters)
            for li in range(L):
                plan.decode(li, q[li], o=o[li], lse=lse[li], scale=m.softmax_scale, stream=s)
    torch.cuda.synchronize()
    rp = Replay(inp)
    ref = [rp.expected(li, inp.q[li]) for li in range(L)]
    for rep in range(3):
        o.zero_()
        lse.zero_()
        g.replay()
        torch.cuda.synchronize()
        for li in range(L):
            eo, el = compare(o[li], lse[li], *ref[li])
            assert eo <= O_TOL and el <= LSE_TOL, (rep, li, eo, el)
    assert plan.workspace_size() <= ws.numel()
    del g
