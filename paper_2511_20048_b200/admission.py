"""Decode-batch composition under an engine capacity cap (S8(f) F4: "SJF speculation-first
batch composition in the bench's batch builder").

PAPER.md:398-422 (Sec. "Inter-Request Schedule"): speculative requests decode fewer than
ten tokens while the main agent requests decode hundreds, so under the engine's default
first-come-first-serve policy short speculative jobs "queued behind long reasoning jobs"
finish too late to be reused; SPAgent instead prioritises speculative requests
("speculation-first", inspired by Short-Job-First).  This module is that rule applied to
one decode step: given the waiting requests and a cap on the batch size, choose which
enter the step.  Host logic only (no device work); the decode step itself is
`spa_decode_plan` + `spa_decode_attention` over the admitted requests.

    fcfs: admit in arrival order.
    sjf:  admit speculative requests first (arrival order), then main requests (arrival
          order) -- ties never reorder requests of the same kind.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Waiting:
    name: object        # the caller's handle (e.g. a request id or a (group, member) pair)
    speculative: bool   # a speculative action request or a main agent request
    arrival: int        # arrival order (smaller = earlier)


def compose_batch(waiting: list[Waiting], max_batch: int, policy: str = "sjf") -> list[object]:
    """Names of the requests admitted to one decode step, in the order they were chosen."""
    if max_batch < 0:
        raise ValueError("max_batch must be >= 0")
    if policy == "fcfs":
        order = sorted(waiting, key=lambda w: w.arrival)
    elif policy == "sjf":
        order = sorted(waiting, key=lambda w: (not w.speculative, w.arrival))
    else:
        raise ValueError(f"unknown policy {policy!r}")
    return [w.name for w in order[:max_batch]]
