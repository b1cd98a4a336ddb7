"""Seeded synthetic batch recipes for the BASELINE.json configs (no method arithmetic).

A recipe describes the *shape* of one decode batch under SPAgent speculation:
agent groups, each with a main (reasoning) request holding context c_i of length P
(Sec. II-A "context c_i containing the system prompt along with all
previous thoughts, actions, and observations"), an optional private reasoning tail,
and k speculative requests that fork from c_i (PAPER.md:189 Aggressive phase: "samples
k speculative actions"; PAPER.md:198 Verified phase: "a parallel speculative path
samples k candidate actions"; "all samples of one request share the same
prefix").  A fork's own tail is a 16-token speculation instruction plus U{1..10}
generated tokens ("typically fewer than ten tokens").

Recipes are consumed by the bench and the GPU tests (driving the C ABI) and by the
oracle (replaying the same call log on its dense model).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Model:
    name: str
    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    page_size: int = 16
    scale: float | None = None  # None -> 1/sqrt(d)

    @property
    def softmax_scale(self) -> float:
        return self.scale if self.scale is not None else self.head_dim ** -0.5


TINY = Model("tiny", 1, 8, 2, 64)
QWEN25_32B = Model("qwen2.5-32b", 64, 40, 8, 128)
# Gemma-3-27B: query_pre_attn_scalar = 168 -> scale 168^-0.5 [EXT: HF Gemma3 config]
GEMMA3_27B = Model("gemma-3-27b", 62, 32, 16, 128, scale=168 ** -0.5)


@dataclass
class Group:
    prefix: int                 # |c_i|, tokens shared by every member
    parent_tail: int | None     # None: no main request in the batch (Aggressive phase)
    fork_tails: list[int] = field(default_factory=list)
    # nested forks (reading #17): a speculative request "s" forks c_i and appends its
    # speculation prompt of spec_prompt tokens (prefilled once); the k samples
    # (fork_tails) then fork from s at prefix + spec_prompt instead of from main at prefix.
    spec_prompt: int | None = None
    spec_in_batch: bool = False   # s itself decodes in the batch (else it only holds the prompt)


@dataclass
class Recipe:
    name: str
    model: Model
    groups: list[Group]
    seed: int
    window: int = 0                 # sliding window of local layers (0 = full)
    local_layers: tuple = ()        # indices of windowed layers (Gemma 5:1 pattern)

    @property
    def n_requests(self) -> int:
        return sum((g.parent_tail is not None) + len(g.fork_tails) for g in self.groups)


def _fork_tail(rng) -> int:
    return 16 + int(rng.integers(1, 11))


def tiny(prefix: int = 256) -> Recipe:
    """BJ config 0: 1 reasoning request + 1 fork sharing a `prefix`-token context."""
    return Recipe("tiny", TINY, [Group(prefix, 8, [4])], seed=0)


def qwen(seed: int = 1, n_agents: int = 32) -> Recipe:
    """BJ config 1: 32 agent trajectories + 32 forks, contexts 2k-8k."""
    rng = np.random.default_rng(seed)
    groups = []
    for _ in range(n_agents):
        p = int(rng.integers(2048, 8193))
        t = int(rng.integers(0, 257))
        groups.append(Group(p, t, [_fork_tail(rng)]))
    return Recipe("qwen2.5-32b", QWEN25_32B, groups, seed=seed)


def gemma(seed: int = 2, n_agents: int = 64) -> Recipe:
    """BJ config 2: 64 agents, 4k-16k contexts, half in Verified phase with k=3 forks."""
    rng = np.random.default_rng(seed)
    groups = []
    for _ in range(n_agents):
        p = int(rng.integers(4096, 16385))
        t = int(rng.integers(0, 257))
        k = 3 if rng.random() < 0.5 else 0
        groups.append(Group(p, t, [_fork_tail(rng) for _ in range(k)]))
    local = tuple(i for i in range(GEMMA3_27B.num_layers) if (i % 6) != 5)
    return Recipe("gemma-3-27b", GEMMA3_27B, groups, seed=seed, window=1024, local_layers=local)


def sweep(batch: int, frac: float, seed: int | None = None) -> Recipe:
    """BJ config 3: batch B, speculative fraction f, Qwen shape."""
    fi = [0.0, 0.25, 0.5, 0.75, 1.0].index(frac) if frac in (0.0, 0.25, 0.5, 0.75, 1.0) else 9
    rng = np.random.default_rng(seed if seed is not None else 3000 + 10 * batch + fi)
    n_fork = int(round(frac * batch))
    groups = []
    if n_fork < batch:
        n_par = batch - n_fork
        tails = [[] for _ in range(n_par)]
        for i in range(n_fork):
            tails[i % n_par].append(_fork_tail(rng))
        for j in range(n_par):
            groups.append(Group(int(rng.integers(2048, 8193)), int(rng.integers(0, 257)), tails[j]))
    else:
        left = batch
        while left > 0:
            k = min(3, left)
            groups.append(Group(int(rng.integers(2048, 8193)), None, [_fork_tail(rng) for _ in range(k)]))
            left -= k
    return Recipe(f"sweep-B{batch}-f{frac}", QWEN25_32B, groups, seed=seed or 3000 + 10 * batch + fi)


def nested(seed: int = 6, n_agents: int = 8, model: Model | None = None, prefix=(2048, 8192), k: int = 3) -> Recipe:
    """Aggressive / Verified phase with nested forks (reading #17):
    each agent's speculative request forks c_i and appends a 16-token speculation prompt, and
    its k samples fork from it and decode U{1..10} tokens.  Agents alternate between the main
    request present (Verified) and absent (Aggressive); every third agent's speculative
    request also decodes."""
    rng = np.random.default_rng(seed)
    groups = []
    for i in range(n_agents):
        p = int(rng.integers(prefix[0], prefix[1] + 1))
        t = int(rng.integers(0, 257)) if i % 2 == 0 else None
        groups.append(Group(p, t, [int(rng.integers(1, 11)) for _ in range(k)], spec_prompt=16,
                            spec_in_batch=i % 3 == 2))
    return Recipe(f"nested-k{k}", model or QWEN25_32B, groups, seed=seed)


def long32k(seed: int = 5, n_agents: int = 128) -> Recipe:
    """BJ config 4: 128 agents with 30k-32k contexts + 1 fork each."""
    rng = np.random.default_rng(seed)
    groups = []
    for _ in range(n_agents):
        p = int(rng.integers(30720, 32769))
        t = int(rng.integers(0, 257))
        groups.append(Group(p, t, [_fork_tail(rng)]))
    return Recipe("long-32k", QWEN25_32B, groups, seed=seed)


def random_small(seed: int, model: Model | None = None, max_prefix: int = 300, nested: bool | None = None) -> Recipe:
    """Random small batches for parity tests: ragged prefixes (aligned and not), tails,
    parent-less groups, nested forks (samples of a speculative request, reading #17),
    multiple KV heads.  nested: None = 30 % of seeds, True / False = force."""
    rng = np.random.default_rng(seed)
    if model is None:
        kv = int(rng.choice([1, 2, 4]))
        g = int(rng.choice([1, 2, 4, 5, 8]))
        d = int(rng.choice([64, 128]))
        model = Model(f"rand{seed}", 2, kv * g, kv, d)
    groups = []
    for _ in range(int(rng.integers(1, 6))):
        p = int(rng.integers(1, max_prefix + 1))
        has_parent = rng.random() < 0.8
        pt = int(rng.integers(0, 40)) if has_parent else None
        nf = int(rng.integers(0 if has_parent else 1, 4))
        groups.append(Group(p, pt, [int(rng.integers(0, 30)) for _ in range(nf)]))
    # nested forks drawn after the flat groups, so earlier seeds keep their batches
    if nested is None:
        nested = rng.random() < 0.3
    if nested:
        for g in groups:
            if g.fork_tails and rng.random() < 0.7:
                g.spec_prompt = int(rng.integers(0, 40))
                g.spec_in_batch = bool(rng.random() < 0.4)
    return Recipe(f"rand{seed}", model, groups, seed=seed)


# ----------------------------------------------------------------------------- call log
def call_log(recipe: Recipe):
    """The ordered allocator calls that build `recipe`'s batch.

    Yields tuples:
      ("alloc", name)                       -> new request named `name`
      ("append", name, origin, start, n)    -> append n tokens at logical positions
                                               [start, start+n) of stream `origin`
      ("fork", child, parent, prefix_len)
    Names are (i, "main") / (i, "s") (nested speculative request) / (i, "f{j}").  A parent-less group still allocates
    and fills its main request (the owner of c_i) but it is not part of the batch.
    `batch` lists the request names of the decode batch, group by group.
    """
    ops = []
    batch = []
    for gi, g in enumerate(recipe.groups):
        main = (gi, "main")
        ops.append(("alloc", main))
        ops.append(("append", main, main, 0, g.prefix))
        src, at = main, g.prefix
        if g.spec_prompt is not None:   # nested: the samples fork from the speculative request
            sp = (gi, "s")
            ops.append(("fork", sp, main, g.prefix))
            if g.spec_prompt:
                ops.append(("append", sp, sp, g.prefix, g.spec_prompt))
            src, at = sp, g.prefix + g.spec_prompt
        for j, ft in enumerate(g.fork_tails):
            ch = (gi, f"f{j}")
            ops.append(("fork", ch, src, at))
            if ft:
                ops.append(("append", ch, ch, at, ft))
        if g.parent_tail:
            ops.append(("append", main, main, g.prefix, g.parent_tail))
        if g.parent_tail is not None:
            batch.append(main)
        if g.spec_prompt is not None and g.spec_in_batch:
            batch.append((gi, "s"))
        batch.extend((gi, f"f{j}") for j in range(len(g.fork_tails)))
    return ops, batch
