"""Pins for oracle/kvmodel.py (CPU only).

Pins: a hand-traced golden call log (tests/golden/paging_trace.json), and a brute-force
physical simulation: every write is tagged with (stream, logical position) into a tiny
pool array using the model's page tables; gathering pool[pt[t // ps]][t % ps] must
reproduce each request's logical token list, where a fork is a plain list copy (the
north_star's "prefix physically copied" reference).  Random call sequences come from
hypothesis.
"""
import json
import os

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle.kvmodel import BAD_REQUEST, INVALID_ARG, NO_PAGES, OK, PagingModel

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paging_trace.json")


def test_golden_paging_trace():
    g = json.load(open(GOLD))
    m = PagingModel(g["num_pages"], g["page_size"])
    for step in g["steps"]:
        op = step["op"]
        if op == "alloc":
            st_, rid = m.alloc()
            assert (st_, rid) == (step["expect_status"], step["expect_id"])
        elif op == "append":
            assert m.append(step["reqs"], step["n"]) == step["expect_status"], step
        elif op == "fork":
            st_, rid = m.fork(step["parent"], step["prefix_len"])
            assert st_ == step["expect_status"], step
            if "expect_id" in step:
                assert rid == step["expect_id"]
        elif op == "free":
            assert m.free(step["req"]) == step["expect_status"]
        for r, (pages, n) in step.get("tables", {}).items():
            st_, t, ln = m.page_table(int(r))
            assert (st_, t, ln) == (OK, pages, n), (step, t, ln)
        for p, c in step.get("refcount", {}).items():
            assert m.refcount[int(p)] == c, step
        if "free" in step:
            assert m.free_pages == step["free"], step
        m.check_invariants()


class PhysicalSim:
    """Tagged physical pool driven by the model's page tables + a plain logical model."""

    def __init__(self, num_pages, ps):
        self.m = PagingModel(num_pages, ps)
        self.ps = ps
        self.pool = [[None] * ps for _ in range(num_pages)]
        self.logical = {}
        self.tag = 0

    def alloc(self):
        st_, r = self.m.alloc()
        self.logical[r] = []
        return r

    def append(self, reqs, ns):
        before = {r: list(self.m.tables.get(r, [])) for r in reqs}
        lens = {r: self.m.lengths.get(r) for r in reqs}
        free_before = self.m.free_pages
        st_ = self.m.append(reqs, ns)
        if st_ != OK:
            for r in reqs:                      # all-or-nothing
                if r in self.m.tables:
                    assert self.m.tables[r] == before[r] and self.m.lengths[r] == lens[r]
            assert self.m.free_pages == free_before
            return st_
        for r, n in zip(reqs, ns):
            for i in range(n):
                pos = lens[r] + i
                page, slot = self.m.slot_of(r, pos)
                self.tag += 1
                self.pool[page][slot] = self.tag
                self.logical[r].append(self.tag)
        return st_

    def fork(self, parent, plen):
        st_, child = self.m.fork(parent, plen)
        if st_ != OK:
            return st_, None
        if plen % self.ps:
            src, dst, rows = self.m.cow_log[-1]
            for s in range(rows):
                self.pool[dst][s] = self.pool[src][s]
        self.logical[child] = list(self.logical[parent][:plen])  # physical copy reference
        return st_, child

    def free(self, r):
        st_ = self.m.free(r)
        if st_ == OK:
            del self.logical[r]
        return st_

    def check(self):
        self.m.check_invariants()
        for r, toks in self.logical.items():
            t = self.m.tables[r]
            gathered = [self.pool[t[i // self.ps]][i % self.ps] for i in range(len(toks))]
            assert gathered == toks, r


ops = st.lists(
    st.tuples(st.sampled_from(["alloc", "append", "append2", "fork", "free"]),
              st.integers(0, 1000), st.integers(0, 1000), st.integers(0, 40)),
    min_size=1, max_size=60)


@settings(max_examples=300, deadline=None)
@given(ops, st.sampled_from([1, 2, 4, 16]), st.integers(1, 24))
def test_paging_matches_physical_copy_reference(seq, ps, num_pages):
    sim = PhysicalSim(num_pages, ps)
    live = []
    for kind, a, b, n in seq:
        if kind == "alloc" or not live:
            live.append(sim.alloc())
        elif kind == "append":
            sim.append([live[a % len(live)]], [n])
        elif kind == "append2" and len(live) >= 2:
            r1, r2 = live[a % len(live)], live[b % len(live)]
            st_ = sim.append([r1, r2], [n, n // 2])
            if r1 == r2:
                assert st_ == INVALID_ARG
        elif kind == "fork":
            p = live[a % len(live)]
            plen = b % (sim.m.lengths[p] + 2)
            st_, c = sim.fork(p, plen)
            if plen > sim.m.lengths[p]:
                assert st_ == INVALID_ARG
            elif st_ == OK:
                live.append(c)
            else:
                assert st_ == NO_PAGES and plen % ps != 0
        elif kind == "free":
            r = live.pop(a % len(live))
            assert sim.free(r) == OK
            assert sim.free(r) == BAD_REQUEST
        sim.check()


def test_lowest_free_id_after_free():
    m = PagingModel(6, 2)
    _, a = m.alloc()
    _, b = m.alloc()
    assert m.append([a, b], [4, 2]) == OK          # a: [0, 1], b: [2]
    assert m.free(a) == OK                          # 0, 1 free again
    _, c = m.alloc()
    assert m.append([c], [1]) == OK
    assert m.page_table(c)[1] == [0]
    assert c == 3                                   # ids never reused


def test_zero_and_full_prefix_forks():
    m = PagingModel(8, 4)
    _, a = m.alloc()
    m.append([a], [6])
    st0, c0 = m.fork(a, 0)
    assert st0 == OK and m.page_table(c0)[1:] == ([], 0)
    st1, c1 = m.fork(a, 6)
    assert st1 == OK and m.page_table(c1)[1] == [0, 2] and m.cow_log[-1] == (1, 2, 2)
    m.check_invariants()


def test_release_window_rule_by_brute_force():
    """P7 pinned by its definition (reading #9): after release_window(W) at length n, every
    key the current query (position n - 1, append-then-attend, reading #8) or a later one
    (keys (q - W, q]) can read lies in a resident page, and every released page holds only
    keys < n - W."""
    for n in range(0, 90, 7):
        for W in (1, 2, 15, 16, 17, 31, 32, 33, 64, 200):
            m = PagingModel(20, 16)
            _, r = m.alloc()
            assert m.append([r], [n]) == 0
            assert m.release_window([r], W) == 0
            t = m.tables[r]
            for q in range(max(0, n - 1), n + 40):      # the current query and later ones
                for key in range(max(0, q + 1 - W), min(q + 1, n)):
                    assert t[key // 16] >= 0, (n, W, q, key)
            for i, p in enumerate(t):
                if p < 0:
                    assert (i + 1) * 16 <= n - W
            m.check_invariants()


def test_release_window_hand_case_and_forks():
    m = PagingModel(20, 16)
    _, r = m.alloc()
    m.append([r], [100])                               # pages 0..6, keys 0..99
    assert m.release_window([r], 32) == 0              # the query at 99 reads keys 68..99
    assert m.tables[r] == [-1, -1, -1, -1, 4, 5, 6]    # pages 0-3 hold keys 0..63 only
    assert m.free_pages == list(range(0, 4)) + list(range(7, 20))
    st, c = m.fork(r, 96)                              # full pages only: -1 entries copied
    assert st == 0 and m.tables[c] == [-1, -1, -1, -1, 4, 5]
    assert m.refcount[4] == m.refcount[5] == 2 and m.refcount[6] == 1
    assert m.fork(r, 40)[0] == 1                       # partial page 2 was released
    assert m.release_window([r], 0) == 1 and m.release_window([999], 5) == 3
    assert m.free(c) == 0 and m.refcount[4] == 1
    m.check_invariants()
