"""Speculation-first batch composition (paper_2511_20048_b200/admission.py)."""
import random

import pytest

from paper_2511_20048_b200.admission import Waiting, compose_batch


def _queue(n_main=10, n_spec=25, seed=0):
    rng = random.Random(seed)
    arrivals = list(range(n_main + n_spec))
    rng.shuffle(arrivals)
    return [Waiting(("m", i), False, arrivals[i]) for i in range(n_main)] + \
           [Waiting(("s", j), True, arrivals[n_main + j]) for j in range(n_spec)]


@pytest.mark.parametrize("cap", [0, 1, 7, 25, 30, 35, 100])
def test_sjf_admits_every_speculative_request_before_any_main(cap):
    q = _queue()
    got = compose_batch(q, cap, "sjf")
    assert len(got) == min(cap, len(q))
    kinds = [n[0] for n in got]
    assert kinds == sorted(kinds, key=lambda k: k != "s")          # all "s" before any "m"
    spec = sorted((w for w in q if w.speculative), key=lambda w: w.arrival)
    main = sorted((w for w in q if not w.speculative), key=lambda w: w.arrival)
    assert got == [w.name for w in (spec + main)[:cap]]            # arrival order within a kind


@pytest.mark.parametrize("cap", [0, 3, 35, 50])
def test_fcfs_is_the_arrival_prefix(cap):
    q = _queue(seed=3)
    got = compose_batch(q, cap, "fcfs")
    assert got == [w.name for w in sorted(q, key=lambda w: w.arrival)][:cap]


def test_same_kind_only_and_errors():
    q = [Waiting(i, True, 10 - i) for i in range(5)]
    assert compose_batch(q, 5, "sjf") == compose_batch(q, 5, "fcfs") == [4, 3, 2, 1, 0]
    with pytest.raises(ValueError):
        compose_batch(q, 2, "lifo")
    with pytest.raises(ValueError):
        compose_batch(q, -1)
