"""Independent models of the KV state: dense logical KV and the paging policy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

LogicalKV is the reference the north_star names: "a forked shared-prefix request equals
the same request with its prefix physically copied".  Each request owns dense arrays;
`fork(parent, P)` copies parent[:P] ("all samples of one request share the
same prefix"; PAPER.md:189 / :198 the k speculative samples are drawn from context c_i).

PagingModel is the documented allocation policy (readings #3, #4, #17),
written independently of the C++ allocator so that page tables, lengths, refcounts and
the free set can be compared bit-exactly ("page-table/fork indexing must match
bit-exactly", BASELINE.json north_star):

  P1  page ids 0..num_pages-1; allocation always takes the LOWEST free id;
  P2  request ids are issued 1, 2, 3, ... and never reused; a freed id is BAD_REQUEST;
  P3  append(reqs, n_new): all-or-nothing -- if the pages needed,
        sum_r ceil((len_r + n_r) / ps) - ceil(len_r / ps),
      exceed the free count the call fails with NO_PAGES and nothing changes;
      otherwise, request by request in list order and token by token, a page is
      allocated exactly when len % ps == 0, and the token goes to slot len % ps of the
      last page;
  P4  fork(parent, P), 0 <= P <= len(parent): the child shares pages [0, floor(P/ps))
      (refcount + 1 each); if P % ps != 0 one fresh page is allocated and slots
      [0, P % ps) of parent page floor(P/ps) are copied into it (copy-on-write at
      fork time, reading #3); child length = P; P > len -> INVALID_ARG;
  P5  free(req): refcount - 1 on every page of the request, pages reaching 0 return to
      the free set;
  P6  invariant: a page with refcount > 1 is full and is never written again.
  P7  release_window(reqs, W) (S8(f) F4, ring-buffer storage for sliding-window layers):
      under append-then-attend (reading #8) the current step's query sits at len - 1 and
      later ones after it; a query at q reads keys (q - W, q] (reading #9), so for each
      listed request the pages i with (i + 1) * ps <= len - W are dead: refcount - 1
      (free at 0) and the table entry becomes -1.  A fork copies -1 entries as -1 (no refcount); a
      fork whose partial page is released is INVALID_ARG.  W <= 0 -> INVALID_ARG.

Status codes mirror include/spa.h: OK 0, INVALID_ARG 1, NO_PAGES 2, BAD_REQUEST 3.
"""
from __future__ import annotations

import heapq

import numpy as np

OK, INVALID_ARG, NO_PAGES, BAD_REQUEST = 0, 1, 2, 3


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


class PagingModel:
    def __init__(self, num_pages: int, page_size: int = 16):
        self.ps = page_size
        self.num_pages = num_pages
        self.refcount = [0] * num_pages
        self._free = list(range(num_pages))  # a min-heap of free page ids (P1)
        heapq.heapify(self._free)
        self.tables: dict[int, list[int]] = {}
        self.lengths: dict[int, int] = {}
        self.next_id = 1                      # P2
        # every physical write, for byte-level checks: (page, slot) <- (req, logical pos)
        self.cow_log: list[tuple[int, int, int]] = []  # (src_page, dst_page, n_rows)

    # -- queries ---------------------------------------------------------------
    @property
    def free_pages(self) -> list[int]:
        return sorted(self._free)

    def page_table(self, req: int):
        if req not in self.tables:
            return BAD_REQUEST, None, None
        return OK, list(self.tables[req]), self.lengths[req]

    def slot_of(self, req: int, pos: int) -> tuple[int, int]:
        """Physical (page, slot) holding logical token `pos` of `req`."""
        return self.tables[req][pos // self.ps], pos % self.ps

    # -- mutations ---------------------------------------------------------------
    def _take(self) -> int:
        p = heapq.heappop(self._free)
        assert self.refcount[p] == 0
        self.refcount[p] = 1
        return p

    def alloc(self):
        rid = self.next_id
        self.next_id += 1
        self.tables[rid] = []
        self.lengths[rid] = 0
        return OK, rid

    def append(self, reqs, n_new):
        if len(reqs) != len(n_new):
            return INVALID_ARG
        if len(set(reqs)) != len(reqs):
            return INVALID_ARG
        for r, n in zip(reqs, n_new):
            if r not in self.tables:
                return BAD_REQUEST
            if n < 0:
                return INVALID_ARG
        need = sum(_cdiv(self.lengths[r] + n, self.ps) - _cdiv(self.lengths[r], self.ps)
                   for r, n in zip(reqs, n_new))
        if need > len(self._free):
            return NO_PAGES                                    # P3 all-or-nothing
        for r, n in zip(reqs, n_new):
            for _ in range(n):
                L = self.lengths[r]
                if L % self.ps == 0:
                    self.tables[r].append(self._take())
                last = self.tables[r][-1]
                assert self.refcount[last] == 1, "P6: write into a shared page"
                self.lengths[r] = L + 1
        return OK

    def fork(self, parent: int, prefix_len: int):
        if parent not in self.tables:
            return BAD_REQUEST, None
        if prefix_len < 0 or prefix_len > self.lengths[parent]:
            return INVALID_ARG, None
        full, rem = divmod(prefix_len, self.ps)
        if rem and not self._free:
            return NO_PAGES, None
        if rem and self.tables[parent][full] < 0:
            return INVALID_ARG, None                            # P7
        st, child = self.alloc()
        shared = self.tables[parent][:full]
        for p in shared:
            if p >= 0:
                self.refcount[p] += 1
        table = list(shared)
        if rem:
            dst = self._take()
            self.cow_log.append((self.tables[parent][full], dst, rem))
            table.append(dst)
        self.tables[child] = table
        self.lengths[child] = prefix_len
        return OK, child

    def free(self, req: int):
        if req not in self.tables:
            return BAD_REQUEST
        for p in self.tables.pop(req):
            if p < 0:
                continue
            self.refcount[p] -= 1
            if self.refcount[p] == 0:
                heapq.heappush(self._free, p)
        del self.lengths[req]
        return OK

    def release_window(self, reqs, window: int):
        if window <= 0:
            return INVALID_ARG
        if any(r not in self.tables for r in reqs):
            return BAD_REQUEST
        for r in reqs:
            t = self.tables[r]
            for i in range(len(t)):
                if (i + 1) * self.ps <= self.lengths[r] - window and t[i] >= 0:
                    self.refcount[t[i]] -= 1
                    if self.refcount[t[i]] == 0:
                        heapq.heappush(self._free, t[i])
                    t[i] = -1
        return OK

    def check_invariants(self):
        """P6 and refcount bookkeeping; raises AssertionError on violation."""
        count = [0] * self.num_pages
        for r, t in self.tables.items():
            assert len(t) == _cdiv(self.lengths[r], self.ps)
            for i, p in enumerate(t):
                if p >= 0:
                    count[p] += 1
        assert count == self.refcount
        free = set(self._free)
        assert len(free) == len(self._free)
        for p in range(self.num_pages):
            assert (p in free) == (count[p] == 0)
        for r, t in self.tables.items():
            for i, p in enumerate(t):
                if p >= 0 and self.refcount[p] > 1:
                    # shared => full for every holder
                    assert self.lengths[r] >= (i + 1) * self.ps


class LogicalKV:
    """Dense per-request K/V (bf16 bit patterns) for a chosen subset of layers."""

    def __init__(self, n_layers_stored: int, n_kv_heads: int, head_dim: int):
        self.L = n_layers_stored
        self.H = n_kv_heads
        self.d = head_dim
        self.K: dict = {}
        self.V: dict = {}

    def alloc(self, name):
        self.K[name] = np.zeros((self.L, 0, self.H, self.d), np.uint16)
        self.V[name] = np.zeros((self.L, 0, self.H, self.d), np.uint16)

    def append(self, name, k_bits: np.ndarray, v_bits: np.ndarray):
        """k_bits, v_bits: [L_stored, n, Hkv, d] uint16."""
        self.K[name] = np.concatenate([self.K[name], k_bits], axis=1)
        self.V[name] = np.concatenate([self.V[name], v_bits], axis=1)

    def fork(self, child, parent, prefix_len: int):
        """Physical copy of the parent's first prefix_len tokens."""
        self.K[child] = self.K[parent][:, :prefix_len].copy()
        self.V[child] = self.V[parent][:, :prefix_len].copy()

    def free(self, name):
        del self.K[name]
        del self.V[name]

    def length(self, name) -> int:
        return self.K[name].shape[1]
