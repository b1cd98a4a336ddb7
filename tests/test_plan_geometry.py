"""Kernel geometry the planner picks (metadata-only pools, CPU only): fp8 pools run 16-row
items as 8 one-warp teams per CTA and 32-row items as 4 teams of one warp per row tile;
bf16 16-row items keep 4 teams of two key-split warps; an explicit teams_per_cta the
one-warp layout does not support keeps the key-split pairs (include/spa.h teams_per_cta;
DESIGN.md S5 "Team geometry")."""
import numpy as np
import pytest

from paper_2511_20048_b200 import spa


def qwen_pool(fp8, num_pages=4096):
    """Qwen2.5-32B attention shape (40 Q / 8 KV heads, d = 128), one layer, no device memory."""
    scale = np.ones((1, 8, 2), np.float32) if fp8 else None
    return spa.Pool(1, 40, 8, 128, num_pages, kv_scale=scale)


@pytest.mark.parametrize("fp8,max_rows,teams,expect", [
    (False, 16, 0, (4, 8)),    # 4 teams x 2 key-split warps
    (True, 16, 0, (8, 8)),     # 8 one-warp teams
    (True, 16, 4, (4, 8)),     # explicit 4 teams: key-split pairs
    (True, 16, 2, (2, 4)),
    (False, 32, 0, (4, 8)),    # one warp per 16-row tile, 4 teams
    (True, 32, 0, (4, 8)),
    (True, 64, 0, (1, 8)),     # 64-row items: 4 tiles x 2 key-split warps
])
def test_geometry(fp8, max_rows, teams, expect):
    pool = qwen_pool(fp8)
    plan = spa.Plan(pool, max_rows=max_rows, teams_per_cta=teams, num_ctas=148)
    nc, tm, wp = plan.geometry()
    assert nc == 148 and (tm, wp) == expect


def test_fp8_auto_rows_takes_32_row_items_for_k3_forks():
    # a parent and 3 forks of one context (k = 3, G = 5: 20 rows > 16) -> 32-row items
    pool = qwen_pool(True)
    parent = pool.alloc()
    pool.append([parent], [2048])
    forks = [pool.fork(parent, 2048) for _ in range(3)]
    for f in forks:
        pool.append([f], [1])
    pool.append([parent], [1])
    plan = spa.Plan(pool, num_ctas=148)
    assert plan.geometry()[1:] == (8, 8)       # before planning: 16-row default
    plan.plan([parent] + forks)
    assert plan.geometry()[1:] == (4, 8)       # 32-row items: 4 teams, one warp per row tile
    assert plan.stats()["rows_max"] == 20


@pytest.mark.parametrize("fp8,window,teams_req,expect", [
    (True, 0, 0, (8, 8)),       # fp8, full attention: 8 one-warp teams
    (True, 256, 0, (12, 12)),   # fp8, windowed: 12 one-warp teams (2-stage rings)
    (True, 256, 4, (4, 8)),     # explicit teams: key-split pairs
    (False, 256, 0, (4, 8)),    # bf16 windowed: key-split pairs
])
def test_windowed_geometry(fp8, window, teams_req, expect):
    pool = qwen_pool(fp8)
    reqs = []
    for n in (700, 1500):
        r = pool.alloc()
        pool.append([r], [n])
        reqs.append(r)
    plan = spa.Plan(pool, max_rows=16, teams_per_cta=teams_req, num_ctas=148)
    plan.plan(reqs, window)
    assert plan.geometry()[1:] == expect
