"""Host planner invariants (metadata-only pools, CPU only).

For every batch row r and KV head h the work descriptors containing r must cover its
attended keys [lo_r, n_r) exactly once (with the member's lower bound applied), read
each key through the right physical page, and the static schedule must run every item
exactly once.  With sharing on, a shared page is read once per (KV head, group).
"""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2511_20048_b200 import spa
from paper_2511_20048_b200.spa import SpaError
from spa_inputs import workloads

DBG_DESC, DBG_MEMBER, DBG_ITEM, DBG_QUEUE, _, DBG_PAGES, DBG_REC_PTR = range(7)


def build(recipe, num_pages=None):
    m = recipe.model
    ops, batch = workloads.call_log(recipe)
    need = sum(-(-(g.prefix + (g.spec_prompt or 0) + max([g.parent_tail or 0] + g.fork_tails)) // 16)
               * (2 + len(g.fork_tails)) for g in recipe.groups) + 16
    pool = spa.Pool(1, m.num_q_heads, m.num_kv_heads, m.head_dim, num_pages or need)
    ids = {}
    for op in ops:
        if op[0] == "alloc":
            ids[op[1]] = pool.alloc()
        elif op[0] == "append":
            pool.append([ids[op[1]]], [op[4]])
        elif op[0] == "fork":
            ids[op[1]] = pool.fork(ids[op[2]], op[3])
    return pool, [ids[n] for n in batch]


def check_plan(pool, plan, reqs, window, n_query=None):
    """Every query row's live keys [lo, hi) are covered exactly once, through the right
    physical pages; rows are request-major, token-minor (spa_extend_plan)."""
    descs = plan.debug_array(DBG_DESC)
    mems = plan.debug_array(DBG_MEMBER)
    items = plan.debug_array(DBG_ITEM)
    queue = plan.debug_array(DBG_QUEUE)
    pages = plan.debug_array(DBG_PAGES)
    rec_ptr = plan.debug_array(DBG_REC_PTR)
    Hkv = pool.cfg.num_kv_heads
    n_query = [1] * len(reqs) if n_query is None else list(n_query)
    row_tab, row_hi = [], []
    for r, nq in zip(reqs, n_query):
        _, tab, n = pool.page_table(r)
        for t in range(nq):
            row_tab.append(tab)
            row_hi.append(n - nq + t + 1)
    N = len(row_tab)
    row_lo = [max(0, h - window) if window > 0 else 0 for h in row_hi]
    cover = [dict() for _ in range(N)]   # token -> count
    occ = [0] * N
    recs = [[] for _ in range(N)]
    tail_owner = {}   # (descriptor, folded page index) -> owning row (one request's rows only)
    for di, d in enumerate(descs):
        page_off, n_pages, t0, t1, moff, nmem, kind, group, n_main = d[:9]
        # shared pages [0, n_main) hold keys [t0, t1); folded member tails follow (reading #21)
        assert t0 % 16 == 0 and t1 <= t0 + 16 * n_main and t1 > t0 + 16 * (n_main - 1)
        for mi in range(moff, moff + nmem):
            row, lo, rec, hi, tk0, tn, ttok, _ = mems[mi]
            occ[row] += 1
            recs[row].append(rec)
            tab = row_tab[row]
            assert lo == row_lo[row] and hi == row_hi[row]
            for t in range(max(t0, lo), min(t1, hi)):
                assert pages[page_off + (t - t0) // 16] == tab[t // 16], "wrong physical page"
                cover[row][t] = cover[row][t] + 1 if t in cover[row] else 1
            if tn:
                assert n_main <= tk0 and tk0 + tn <= n_pages and ttok % 16 == 0 and ttok >= t1
                for k in range(tk0, tk0 + tn):   # a folded page belongs to one request
                    prev = tail_owner.setdefault((di, k), row)
                    assert prev == row or row_tab[prev] is tab
                for t in range(max(ttok, lo), min(ttok + 16 * tn, hi)):
                    assert pages[page_off + tk0 + (t - ttok) // 16] == tab[t // 16], "wrong folded page"
                    cover[row][t] = cover[row][t] + 1 if t in cover[row] else 1
        assert all((di, k) in tail_owner for k in range(n_main, n_pages)), "a folded page nobody owns"
    for r in range(N):
        assert sorted(cover[r]) == list(range(row_lo[r], row_hi[r])), r
        assert all(c == 1 for c in cover[r].values())
        if occ[r] == 1:
            assert recs[r] == [-1] and rec_ptr[r + 1] == rec_ptr[r]
        else:
            assert sorted(recs[r]) == list(range(rec_ptr[r], rec_ptr[r + 1]))
    assert len(items) == len(descs) * Hkv
    assert sorted((a, b) for a, b in items) == sorted((d, h) for d in range(len(descs)) for h in range(Hkv))
    assert sorted(queue) == list(range(len(items)))
    costs = [descs[items[i][0]][1] for i in queue]
    assert all(a >= b for a, b in zip(costs, costs[1:])), "queue must pop the largest items first"

    return descs, mems


@settings(max_examples=80, deadline=None)
@given(st.integers(0, 100_000), st.sampled_from([0, 0, 1, 7, 16, 40, 300]), st.booleans(),
       st.sampled_from([16, 32]), st.sampled_from([0, 1, 3]))
def test_random_batches_cover_every_key_once(seed, window, sharing, max_rows, split):
    rec = workloads.random_small(seed)
    pool, reqs = build(rec)
    G = rec.model.num_q_heads // rec.model.num_kv_heads
    if G > max_rows:
        return
    plan = spa.Plan(pool, sharing=sharing, max_rows=max_rows, split_pages=split, num_ctas=3)
    plan.plan(reqs, window)
    check_plan(pool, plan, reqs, window)


def test_shared_prefix_read_once_per_group_and_head():
    rec = workloads.qwen(seed=1)
    pool, reqs = build(rec)
    plan = spa.Plan(pool, num_ctas=148)
    plan.plan(reqs)
    descs, mems = check_plan(pool, plan, reqs, 0)
    s = plan.stats()
    # every group: one parent + one fork with a >= 2048-token shared prefix
    assert s["n_groups"] == 32 and s["rows_max"] == 10
    shared_tokens = sum(g.prefix // 16 * 16 for g in rec.groups)
    tail_tokens = sum(g.prefix % 16 * 2 + g.parent_tail + g.fork_tails[0] for g in rec.groups)
    assert s["unique_tokens"] == shared_tokens + tail_tokens
    assert s["unshared_tokens"] == sum(2 * g.prefix + g.parent_tail + g.fork_tails[0] for g in rec.groups)
    assert s["unshared_tokens"] / s["unique_tokens"] > 1.9


def test_sharing_off_is_groups_of_one():
    rec = workloads.qwen(seed=1, n_agents=4)
    pool, reqs = build(rec)
    plan = spa.Plan(pool, sharing=False, num_ctas=8)
    plan.plan(reqs)
    descs, _ = check_plan(pool, plan, reqs, 0)
    assert all(d[5] == 1 for d in descs)
    s = plan.stats()
    assert s["unique_tokens"] == s["unshared_tokens"]


def test_subgroups_when_rows_exceed_max_rows():
    rec = workloads.sweep(16, 0.75)         # parents with 3 forks: 4 x 5 = 20 rows
    pool, reqs = build(rec)
    p16 = spa.Plan(pool, max_rows=16, num_ctas=4)
    p16.plan(reqs)
    p32 = spa.Plan(pool, max_rows=32, num_ctas=4)
    p32.plan(reqs)
    check_plan(pool, p16, reqs, 0)
    check_plan(pool, p32, reqs, 0)
    assert p16.stats()["rows_max"] <= 16 and p32.stats()["rows_max"] == 20
    assert p32.stats()["unique_tokens"] < p16.stats()["unique_tokens"]


def test_window_restricts_to_union_of_windows():
    rec = workloads.gemma(seed=2, n_agents=6)
    pool, reqs = build(rec)
    plan = spa.Plan(pool, num_ctas=16)
    plan.plan(reqs, window=1024)
    check_plan(pool, plan, reqs, 1024)
    s = plan.stats()
    assert s["unshared_tokens"] == 1024 * len(reqs)


def test_plan_errors():
    pool = spa.Pool(1, 4, 2, 64, 8)
    a = pool.alloc()
    b = pool.alloc()
    pool.append([a], [5])
    plan = spa.Plan(pool)
    with pytest.raises(SpaError) as e:
        plan.plan([a, a])
    assert e.value.status == spa.SPA_ERR_INVALID_ARG
    with pytest.raises(SpaError) as e:
        plan.plan([a, b])                 # b is empty
    assert e.value.status == spa.SPA_ERR_INVALID_ARG
    with pytest.raises(SpaError) as e:
        plan.plan([a, 999])
    assert e.value.status == spa.SPA_ERR_BAD_REQUEST
    with pytest.raises(SpaError) as e:
        spa.Plan(pool, max_rows=24)
    assert e.value.status == spa.SPA_ERR_UNSUPPORTED


def test_lpt_schedule_is_balanced():
    rec = workloads.qwen(seed=1)
    pool, reqs = build(rec)
    plan = spa.Plan(pool, num_ctas=148)
    plan.plan(reqs)
    descs = plan.debug_array(DBG_DESC)
    items = plan.debug_array(DBG_ITEM)
    queue = plan.debug_array(DBG_QUEUE)
    import heapq
    teams = [(0, t) for t in range(plan.stats()["n_teams"])]     # greedy list scheduling = the kernel's
    for i in queue:                                              # dynamic queue at equal team speed
        load, t = heapq.heappop(teams)
        heapq.heappush(teams, (load + descs[items[i][0]][1] + 1, t))
    loads = [l for l, _ in teams]
    assert max(loads) <= 1.15 * np.mean(loads)


@settings(max_examples=60, deadline=None)
@given(st.integers(0, 100_000), st.sampled_from([0, 0, 5, 16, 40]), st.booleans(),
       st.sampled_from([16, 32, 64]), st.sampled_from([0, 1, 3]))
def test_extend_batches_cover_every_key_once(seed, window, sharing, max_rows, split):
    """F2: requests contribute their last n_query tokens as causal query rows."""
    rec = workloads.random_small(seed)
    pool, reqs = build(rec)
    G = rec.model.num_q_heads // rec.model.num_kv_heads
    if G > max_rows:
        return
    rng = np.random.default_rng(seed)
    n_query = [int(rng.integers(1, min(pool.page_table(r)[2], 40) + 1)) for r in reqs]
    plan = spa.Plan(pool, sharing=sharing, max_rows=max_rows, split_pages=split, num_ctas=3)
    plan.plan(reqs, window, n_query=n_query)
    check_plan(pool, plan, reqs, window, n_query)
    assert plan.stats()["n_req"] == sum(n_query)


def test_extend_rows_share_the_prefix():
    """A fork's speculative prompt (16 query tokens) and its parent's decode token: the
    parent/fork common prefix is read once per KV head and sub-group of max_rows rows."""
    rec = workloads.qwen(seed=1, n_agents=4)
    pool, reqs = build(rec)
    n_query = [1 if i % 2 == 0 else 16 for i in range(len(reqs))]   # batch = parent, fork, ...
    p64 = spa.Plan(pool, max_rows=64, num_ctas=8)
    p64.plan(reqs, 0, n_query=n_query)
    check_plan(pool, p64, reqs, 0, n_query)
    p16 = spa.Plan(pool, max_rows=16, num_ctas=8)
    p16.plan(reqs, 0, n_query=n_query)
    check_plan(pool, p16, reqs, 0, n_query)
    # 17 rows x G=5 = 85 rows: 2 sub-groups at 64 rows, 6 at 16 -> shared prefix read 2 vs 6 times
    shared = sum(g.prefix // 16 * 16 for g in rec.groups)
    assert p64.stats()["unique_tokens"] < p16.stats()["unique_tokens"]
    assert p64.stats()["unique_tokens"] >= 2 * shared


def test_extend_plan_errors():
    pool = spa.Pool(1, 4, 2, 64, 8)
    a = pool.alloc()
    pool.append([a], [5])
    plan = spa.Plan(pool)
    for bad in ([0], [6], [-1]):
        with pytest.raises(SpaError) as e:
            plan.plan([a], n_query=bad)
        assert e.value.status == spa.SPA_ERR_INVALID_ARG
    plan.plan([a], n_query=[5])
    assert plan.stats()["n_req"] == 5


def test_window_release_bounds_a_local_layer_pool():
    """F4 ring buffer, host side: a Gemma-shaped local-layer pool (W = 1024) that releases
    after every decode step holds about W/16 + 2 pages per request instead of len/16."""
    from spa_inputs import workloads as wl

    rec = wl.gemma(seed=2, n_agents=8)
    pool = spa.Pool(1, 32, 16, 128, 40000)                 # metadata only
    ops, batch = wl.call_log(rec)
    ids = {}
    for op in ops:
        if op[0] == "alloc":
            ids[op[1]] = pool.alloc()
        elif op[0] == "append":
            pool.append([ids[op[1]]], [op[4]])
        elif op[0] == "fork":
            ids[op[1]] = pool.fork(ids[op[2]], op[3])
    reqs = [ids[n] for n in batch]
    used_full = pool.num_pages - len(pool.free_pages())
    W = 1024
    pool.release_window(list(ids.values()), W)
    for _ in range(40):
        pool.append(reqs, [1] * len(reqs))
        pool.release_window(list(ids.values()), W)
        plan = spa.Plan(pool)
        plan.plan(reqs, W)
    used = pool.num_pages - len(pool.free_pages())
    resident = [sum(p >= 0 for p in pool.page_table(i)[1]) for i in ids.values()]
    assert max(resident) <= W // 16 + 2
    assert used < used_full / 4


def test_release_keeps_prefix_sharing_within_a_family():
    """After spa_kv_release_window a parent and its forks release different leading pages
    (their lengths differ); the planner still groups them and reads their common window
    region once, plus a small head range for the member whose window starts earlier."""
    pool = spa.Pool(1, 8, 2, 128, 400)
    parent = pool.alloc()
    pool.append([parent], [600])
    forks = [pool.fork(parent, 600) for _ in range(3)]
    pool.append(forks, [20, 25, 30])
    pool.append([parent], [5])
    reqs = [parent] + forks
    W = 200
    pool.release_window(reqs, W)
    assert len({pool.page_table(r)[1].count(-1) for r in reqs}) > 1     # different release points
    on, off = spa.Plan(pool), spa.Plan(pool, sharing=False)
    on.plan(reqs, W)
    off.plan(reqs, W)
    s_on, s_off = on.stats(), off.stats()
    assert s_on["n_groups"] == 1 and s_off["n_groups"] == 4
    assert s_on["unshared_tokens"] == s_off["unique_tokens"] == 4 * W
    # the common region [max first resident key, 600) is read once instead of 4 times
    assert s_on["unique_tokens"] < 0.5 * s_off["unique_tokens"]


def test_release_family_grouping_with_parent_first_in_batch():
    """The parent (listed first, longest) releases the most pages; forks link to it through
    the pages they still share."""
    pool = spa.Pool(1, 8, 2, 128, 200)
    parent = pool.alloc()
    pool.append([parent], [333])
    forks = [pool.fork(parent, 333) for _ in range(2)]
    pool.append(forks, [17, 19])
    pool.append([parent], [40])
    reqs = [parent] + forks
    pool.release_window(reqs, 200)
    plan = spa.Plan(pool)
    plan.plan(reqs, 200)
    assert plan.stats()["n_groups"] == 1


def test_release_in_documented_order_never_breaks_the_plan():
    """the documented per-step order -- append one token, release_window(W),
    plan(W) -- must never leave the current query (at n - 1, append-then-attend, reading
    #8) reaching a released page.  The old rule (16p + 16 <= n + 1 - W) failed every 16th
    step; the oracle's P7 is the same rule (oracle/kvmodel.py)."""
    W = 100
    pool = spa.Pool(1, 8, 2, 128, 64)
    r = pool.alloc()
    pool.append([r], [1])
    for n in range(2, 400):
        pool.append([r], [1])
        pool.release_window([r], W)
        plan = spa.Plan(pool)
        plan.plan([r], W)          # raises SpaError if the window needs a released page
        t = pool.page_table(r)[1]
        assert all(t[k // 16] >= 0 for k in range(max(0, n - W), n)), n
        assert sum(p >= 0 for p in t) <= W // 16 + 2


def _alg_tokens_brute_force(pool, reqs, window, n_query=None):
    """Distinct (physical page, slot) keys the batch rows attend to (SURVEY.md Sec. 8(d)
    B_alg per KV head), counted from the page tables alone."""
    n_query = [1] * len(reqs) if n_query is None else n_query
    seen = set()
    for r, nq in zip(reqs, n_query):
        _, tab, n = pool.page_table(r)
        for t in range(nq):
            hi = n - nq + t + 1
            lo = max(0, hi - window) if window > 0 else 0
            seen.update((tab[k // 16], k % 16) for k in range(lo, hi))
    return len(seen)


def test_nested_forks_read_each_shared_run_once():
    """Aggressive / Verified shapes with nested forks (reading #17):
    c_i is one range holding every member's rows, the speculative prompt's pages one range
    holding the samples (and the speculative request when it decodes), tails per request."""
    rec = workloads.nested(seed=6, n_agents=6, model=workloads.Model("m", 1, 8, 2, 128), prefix=(300, 700))
    pool, reqs = build(rec)
    ops, batch = workloads.call_log(rec)
    plan = spa.Plan(pool, max_rows=32, num_ctas=4, split_pages=1000)
    plan.plan(reqs)
    descs, mems = check_plan(pool, plan, reqs, 0)
    rows_of = {nm: i for i, nm in enumerate(batch)}
    for gi, g in enumerate(rec.groups):
        members = {rows_of[nm] for nm in batch if nm[0] == gi}
        samples = {rows_of[nm] for nm in batch if nm[0] == gi and nm[1] not in ("main",)}
        ds = [set(mems[mi][0] for mi in range(d[4], d[4] + d[5])) for d in descs]
        # one descriptor holds every member and covers all full pages of c_i
        full = [d for d, m in zip(descs, ds) if m == members]
        assert len(full) == 1 and full[0][2] == 0 and full[0][3] >= g.prefix // 16 * 16
        # the samples (+ s) share the page of s that holds the tail of c_i and the prompt head
        if len(samples) > 1 and g.parent_tail is not None:
            assert any(m == samples for m in ds)
    s = plan.stats()
    assert s["alg_tokens"] == _alg_tokens_brute_force(pool, reqs, 0)
    assert s["unique_tokens"] == s["alg_tokens"]        # nothing read twice at max_rows 32


@settings(max_examples=60, deadline=None)
@given(st.integers(0, 100_000), st.sampled_from([0, 0, 5, 40, 300]), st.sampled_from([16, 32, 64]))
def test_nested_random_batches_cover_every_key_once(seed, window, max_rows):
    rec = workloads.random_small(seed, nested=True)
    pool, reqs = build(rec)
    G = rec.model.num_q_heads // rec.model.num_kv_heads
    if G > max_rows:
        return
    plan = spa.Plan(pool, max_rows=max_rows, split_pages=int(seed % 4), num_ctas=3)
    plan.plan(reqs, window)
    check_plan(pool, plan, reqs, window)
    s = plan.stats()
    assert s["alg_tokens"] == _alg_tokens_brute_force(pool, reqs, window)
    assert s["alg_tokens"] <= s["unique_tokens"] <= s["unshared_tokens"]


def test_alg_tokens_counts_each_key_once_when_a_class_is_chunked():
    """k = 3 on Qwen (G = 5): parent + 3 forks = 20 rows > 16, so c_i is read by two chunks at
    max_rows 16; the algorithmic bytes still count it once (VERDICT r1 roofline accounting)."""
    rec = workloads.sweep(16, 0.75)
    pool, reqs = build(rec)
    p16 = spa.Plan(pool, max_rows=16, num_ctas=4)
    p16.plan(reqs)
    s = p16.stats()
    assert s["alg_tokens"] == _alg_tokens_brute_force(pool, reqs, 0)
    assert s["unique_tokens"] > 1.5 * s["alg_tokens"]
