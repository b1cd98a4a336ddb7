"""fp64 CPU oracle for SPAgent's shared-prefix paged GQA decode-attention step.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` leg (and its `--impl reference` arm) may import, call or execute
anything in this package.  The product path (`paper_2511_20048_b200`) never imports it
and shares no code, header, table or helper with it; the two meet only through the
seeded input generators in `spa_inputs`, which hold none of the method's arithmetic.

Contents
  attention.py  decode attention, written as its plain definition (softmax(scale q K^T) V
                per query head, GQA head mapping, optional sliding window), the causal
                extend (prefill of a request's last T tokens) as that definition per
                token, and the split-KV log-sum-exp merge.
  kvmodel.py    a dense logical KV model (a fork is a physical copy) plus an independent
                model of the documented paging policy (lowest-free page id, refcounts,
                copy-on-write of the partial last page).
  fp8.py        the e4m3 KV quantiser and dequantiser of the FP8-page variant (S8(f) F4),
                from the format definition (round to nearest even, saturating).
  replay.py     replays a batch's allocator call log on the models above and evaluates
                the expected outputs (optionally on FP8-quantised K/V).

Where the paper is silent (it never mentions attention, KV caches or pages -- see
SURVEY.md Sec. 0.1) the readings used here are listed in DESIGN.md Sec. 3 and cited
by number ("reading #k") in the docstrings.

Parity status: every function here is pinned by `tests/test_oracle_*.py` against
closed forms, brute force, a library routine (torch SDPA in fp64) or hand-derived
golden fixtures (`tests/golden/`); none is "parity unpinned".
"""
