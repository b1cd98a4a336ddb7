"""The C++ allocator (metadata-only pool, no GPU) vs the independent oracle paging model.

Page tables, lengths, refcounts, the free set and every status code must match
bit-exactly after every call ("page-table/fork indexing must match bit-exactly",
BASELINE.json north_star).  Drivers: the hand-traced golden log and hypothesis
state machines over random call sequences.
"""
import json
import os

from hypothesis import given, settings
from hypothesis import strategies as st
from hypothesis.stateful import RuleBasedStateMachine, invariant, precondition, rule

from oracle.kvmodel import PagingModel
from paper_2511_20048_b200 import spa

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paging_trace.json")


def _state_equal(pool: spa.Pool, model: PagingModel):
    assert pool.free_pages() == model.free_pages
    assert pool.refcounts() == model.refcount
    for rid in model.tables:
        st_, pages, n = pool.page_table(rid)
        assert (st_, pages, n) == (0, model.tables[rid], model.lengths[rid]), rid


def test_golden_trace_through_library():
    g = json.load(open(GOLD))
    pool = spa.Pool(1, 2, 1, 64, g["num_pages"], page_size=g["page_size"])
    model = PagingModel(g["num_pages"], g["page_size"])
    for step in g["steps"]:
        op = step["op"]
        if op == "alloc":
            rid = pool.alloc()
            _, mid = model.alloc()
            assert rid == mid == step["expect_id"]
        elif op == "append":
            assert pool.append(step["reqs"], step["n"], check=False) == step["expect_status"]
            model.append(step["reqs"], step["n"])
        elif op == "fork":
            st_, child = pool.fork(step["parent"], step["prefix_len"], check=False)
            mst, mchild = model.fork(step["parent"], step["prefix_len"])
            assert st_ == mst == step["expect_status"]
            if st_ == 0:
                assert child == mchild == step["expect_id"]
        elif op == "free":
            assert pool.free(step["req"], check=False) == step["expect_status"]
            model.free(step["req"])
        for r, (pages, n) in step.get("tables", {}).items():
            assert pool.page_table(int(r)) == (0, pages, n)
        _state_equal(pool, model)


class AllocatorMachine(RuleBasedStateMachine):
    def __init__(self):
        super().__init__()
        self.ps = 16
        self.num_pages = 40
        self.pool = spa.Pool(2, 4, 2, 64, self.num_pages, page_size=self.ps)
        self.model = PagingModel(self.num_pages, self.ps)
        self.ids = []      # every id ever issued (freed ones included: BAD_REQUEST paths)

    @rule()
    def alloc(self):
        rid = self.pool.alloc()
        _, mid = self.model.alloc()
        assert rid == mid
        self.ids.append(rid)

    @precondition(lambda self: self.ids)
    @rule(data=st.data())
    def append(self, data):
        k = data.draw(st.integers(1, 3))
        reqs = [data.draw(st.sampled_from(self.ids)) for _ in range(k)]
        ns = [data.draw(st.integers(0, 70)) for _ in range(k)]
        assert self.pool.append(reqs, ns, check=False) == self.model.append(reqs, ns)

    @precondition(lambda self: self.ids)
    @rule(data=st.data())
    def fork(self, data):
        parent = data.draw(st.sampled_from(self.ids))
        ln = self.model.lengths.get(parent, 5)
        plen = data.draw(st.integers(-1, ln + 2))
        st_, child = self.pool.fork(parent, plen, check=False)
        mst, mchild = self.model.fork(parent, plen)
        assert st_ == mst
        if st_ == 0:
            assert child == mchild
            self.ids.append(child)

    @precondition(lambda self: self.ids)
    @rule(data=st.data())
    def free(self, data):
        rid = data.draw(st.sampled_from(self.ids))
        assert self.pool.free(rid, check=False) == self.model.free(rid)

    @precondition(lambda self: self.ids)
    @rule(data=st.data())
    def release_window(self, data):
        k = data.draw(st.integers(1, 3))
        reqs = [data.draw(st.sampled_from(self.ids)) for _ in range(k)]
        w = data.draw(st.sampled_from([0, 1, 15, 16, 17, 40, 100]))
        assert self.pool.release_window(reqs, w, check=False) == self.model.release_window(reqs, w)

    @invariant()
    def same_state(self):
        _state_equal(self.pool, self.model)
        self.model.check_invariants()


TestAllocatorMachine = AllocatorMachine.TestCase
TestAllocatorMachine.settings = settings(max_examples=150, stateful_step_count=40, deadline=None)


@settings(max_examples=60, deadline=None)
@given(st.integers(0, 10_000))
def test_workload_call_logs_match(seed):
    """Replaying a random agent-batch call log gives identical page tables."""
    from spa_inputs import workloads

    rec = workloads.random_small(seed)
    ops, batch = workloads.call_log(rec)
    pool = spa.Pool(1, 4, 2, 64, 400)
    model = PagingModel(400, 16)
    ids = {}
    for op in ops:
        if op[0] == "alloc":
            ids[op[1]] = pool.alloc()
            assert model.alloc()[1] == ids[op[1]]
        elif op[0] == "append":
            r = ids[op[1]]
            assert pool.append([r], [op[4]], check=False) == model.append([r], [op[4]])
        elif op[0] == "fork":
            c = pool.fork(ids[op[2]], op[3])
            assert model.fork(ids[op[2]], op[3]) == (0, c)
            ids[op[1]] = c
    _state_equal(pool, model)
