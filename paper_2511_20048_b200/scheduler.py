"""SPAgent's speculation scheduler driven by measured B200 costs.

Host logic, no GPU work: the cost model of the paper's Sec. IV-A (Eqs. 1-4,
/root/reference/PAPER.md:311-340) with SPEC.md's affine-plus-knee form of the engine's
hybrid-batch time T_h, its least-squares calibration on a measured
profile table (the `prefill_len,prefill_count,decode_count,seconds`
table scripts/th_table.py writes from this library's kernels), and Algorithm 1,
"Runtime Speculation Selection".

One extension over SPEC's model (reading F3-a): a speculative decode request
forked copy-free from its agent's context c_i does not cost what an independent request
costs -- with prefix sharing its attention reads only its own tail ("all
samples of one request share the same prefix") -- so T_h carries a separate per-fork
slope `decode_cost_per_fork` (gamma_f).  Eq. 3's k|S| added decode requests are forks
(P:189), charged gamma_f; gamma_f = None means gamma_f = gamma (SPEC's model, and
the no-sharing control).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field


@dataclass
class CostModelParams:
    """T_h parameters.  Seconds unless stated."""
    base_step_time: float = 0.020          # d0
    decode_cost_per_request: float = 1e-4  # gamma
    decode_knee: float = 64                # N0 (requests)
    decode_slowdown: float = 0.2           # alpha
    prefill_fixed_cost: float = 0.002
    prefill_cost_per_token: float = 5e-5
    decode_cost_per_fork: float | None = None   # gamma_f (reading F3-a); None = gamma

    def __post_init__(self):
        vals = [self.base_step_time, self.decode_cost_per_request, self.decode_knee, self.decode_slowdown,
                self.prefill_fixed_cost, self.prefill_cost_per_token]
        if self.decode_cost_per_fork is not None:
            vals.append(self.decode_cost_per_fork)
        if any(v < 0 for v in vals) or not self.base_step_time > 0:
            raise ValueError("cost model parameters must be >= 0 and base_step_time > 0 (SPEC.md:108)")

    @property
    def gamma_f(self) -> float:
        return self.decode_cost_per_request if self.decode_cost_per_fork is None else self.decode_cost_per_fork


def _decode_term(n: float, g: float, p: CostModelParams) -> float:
    """gamma N for N <= N0, gamma N0 + gamma (1 + alpha)(N - N0) beyond the knee."""
    if n <= p.decode_knee:
        return g * n
    return g * p.decode_knee + g * (1.0 + p.decode_slowdown) * (n - p.decode_knee)


def hybrid_batch_time(prefill, decode_count: float, params: CostModelParams, fork_count: float = 0) -> float:
    """T_h(P, N) (Table I "Engine profiling timing results for hybrid batches";
    SPEC.md:116-124): d0 + decode term + sum over prefill entries (length, count) of
    count (prefill_fixed + per_token length).  fork_count forked decode requests add
    gamma_f each, on the same knee-shaped curve (reading F3-a)."""
    if decode_count < 0 or fork_count < 0:
        raise ValueError("decode_count and fork_count must be >= 0")
    t = params.base_step_time
    # main requests first, then the forks: a request past the knee N0 costs (1 + alpha) x
    # its slope (with gamma_f = gamma this is SPEC's decode term of N + fork_count)
    t += _decode_term(decode_count, params.decode_cost_per_request, params)
    below = max(0.0, min(fork_count, params.decode_knee - decode_count))
    t += params.gamma_f * below + params.gamma_f * (1.0 + params.decode_slowdown) * (fork_count - below)
    for length, count in (prefill or ()):
        t += count * (params.prefill_fixed_cost + params.prefill_cost_per_token * length)
    return t


def decode_overhead(spec_count: int, k: int, n: int, l_s: float, params: CostModelParams) -> float:
    """Eq. 3: T_od = l_s (T_h(emptyset, N + k|S|) - T_h(emptyset, N)); the k|S|
    added decode requests are forks of their agents' contexts (charged gamma_f)."""
    if spec_count == 0:
        return 0.0
    return l_s * (hybrid_batch_time((), n, params, fork_count=k * spec_count) - hybrid_batch_time((), n, params))


def prefill_overhead(spec_count: int, L_s: float, n: int, params: CostModelParams) -> float:
    """Eq. 4: T_op = T_h((L_s, |S|), N) - T_h(emptyset, N), once per selected
    request ("all samples of one request share the same prefix")."""
    if spec_count == 0:
        return 0.0
    return hybrid_batch_time([(L_s, spec_count)], n, params) - hybrid_batch_time((), n, params)


@dataclass
class SpecCandidate:
    """A main request whose k speculative samples have not been launched."""
    task_id: int
    step_index: int
    enqueue_time: float
    wait_time: float = 0.0
    p: float = 0.4          # estimated hit probability (Fig. 1b "overall average of 40%")
    t_act: float = 1.5      # seconds
    L_s: float = 512        # speculative prefill tokens
    l_s: float = 8          # speculative output tokens


def expected_reduction(S, n_m: int, n_a: int, k: int) -> float:
    """Eq. 2: (1 / (N_m + N_a)) sum_{r in S} t_act (1 - (1 - p)^k)."""
    if n_m + n_a <= 0:
        raise ValueError("N_m + N_a must be >= 1 (Eq. 2 denominator)")
    return sum(c.t_act * (1.0 - (1.0 - c.p) ** k) for c in S) / (n_m + n_a)


@dataclass
class GainBreakdown:
    reduction: float
    decode_overhead: float
    prefill_overhead: float

    @property
    def net(self) -> float:
        """Eq. 1: T_r = T_ra - (T_od + T_op)."""
        return self.reduction - (self.decode_overhead + self.prefill_overhead)


def net_gain(S, load, params: CostModelParams, k: int) -> GainBreakdown:
    """Eqs. 1-4 for a selection S at load (N, N_m, N_s, N_a).  l_s and L_s are the
    selection's means (the paper's per-system averages, Table I)."""
    n, n_m, _n_s, n_a = load
    if not S:
        return GainBreakdown(0.0, 0.0, 0.0)
    l_s = sum(c.l_s for c in S) / len(S)
    L_s = sum(c.L_s for c in S) / len(S)
    return GainBreakdown(expected_reduction(S, n_m, n_a, k), decode_overhead(len(S), k, n, l_s, params),
                         prefill_overhead(len(S), L_s, n, params))


def priority_key(c: SpecCandidate):
    """Earlier step first; among equal steps the more recently arrived first; then task id
    (SPEC.md:449-456)."""
    return (c.step_index, -c.enqueue_time, c.task_id)


@dataclass
class SchedulerConfig:
    k: int = 3
    t_w: float = 1.0        # seconds


@dataclass
class SelectResult:
    selected: list
    expired: list
    returned: list = field(default_factory=list)   # the break candidate, back to the queue
    best: float = 0.0


def select_step(queue, load, params: CostModelParams, config: SchedulerConfig) -> SelectResult:
    """Algorithm 1 exactly: pop the highest-priority candidate; drop it if
    its wait exceeds t_w (line 6-7, "Continue"); accept it iff T_r(S + c, N) > T_r,best
    (line 9), else stop (line 13, "Break").  `queue` (a list) is consumed in priority order;
    unpopped candidates and the break candidate stay in it."""
    queue.sort(key=priority_key)
    S, expired = [], []
    best = 0.0
    res = SelectResult(S, expired)
    while queue:
        c = queue.pop(0)
        if c.wait_time > config.t_w:
            expired.append(c)
            continue
        cur = net_gain(S + [c], load, params, config.k).net
        if cur > best:
            best = cur
            S.append(c)
        else:
            queue.insert(0, c)
            res.returned.append(c)
            break
    res.best = best
    return res


# ----------------------------------------------------------------------------- calibration
class CalibrationError(ValueError):
    pass


def _lstsq(rows, y):
    """Least squares by the normal equations (small, well-scaled systems); returns x."""
    n = len(rows[0])
    A = [[sum(r[i] * r[j] for r in rows) for j in range(n)] for i in range(n)]
    b = [sum(r[i] * yy for r, yy in zip(rows, y)) for i in range(n)]
    # Gaussian elimination with partial pivoting
    for c in range(n):
        piv = max(range(c, n), key=lambda r: abs(A[r][c]))
        if abs(A[piv][c]) < 1e-300:
            raise CalibrationError("profile table does not determine the cost model (singular fit)")
        A[c], A[piv] = A[piv], A[c]
        b[c], b[piv] = b[piv], b[c]
        for r in range(c + 1, n):
            f = A[r][c] / A[c][c]
            for j in range(c, n):
                A[r][j] -= f * A[c][j]
            b[r] -= f * b[c]
    x = [0.0] * n
    for c in reversed(range(n)):
        x[c] = (b[c] - sum(A[c][j] * x[j] for j in range(c + 1, n))) / A[c][c]
    return x


def calibrate(table, max_rel_err: float = 0.10, relative: bool = False):
    """Least-squares fit of the T_h parameters on a profile table.
    relative=True minimises relative instead of absolute residuals (each row weighted by
    1 / seconds; reading F3-b): a measured table spanning 1 to 256 decode requests
    covers two orders of magnitude of step time, where absolute least squares leaves the
    small batches with large relative errors.

    table: rows (prefill_len, prefill_count, decode_count, seconds[, fork_count]).  The
    knee N0 is chosen among the table's decode counts (and "no knee") by residual; for each
    N0 the model is linear in (d0, gamma, gamma alpha, prefill_fixed, per_token[, gamma_f]).
    Returns (params, report); raises CalibrationError if the table is underdetermined
    (fewer than 6 rows, or no decode-only / no hybrid rows) or a row is off by more than
    max_rel_err."""
    rows = [tuple(r) + (0,) * (5 - len(r)) for r in table]
    if len(rows) < 6:
        raise CalibrationError(f"profile table has {len(rows)} rows; >= 6 spanning decode-only and hybrid batches needed")
    if not any(r[1] == 0 for r in rows) or not any(r[1] > 0 for r in rows):
        raise CalibrationError("profile table needs decode-only rows (prefill_count 0) and hybrid rows")
    with_forks = any(r[4] > 0 for r in rows)
    if with_forks and not any(r[4] == 0 for r in rows):
        raise CalibrationError("fork rows need fork-free rows beside them to separate gamma from gamma_f")
    best = None
    knees = sorted({float(r[2]) for r in rows}) + [math.inf]
    for n0 in knees:
        X, y = [], []
        for (pl, pc, nd, sec, nf) in rows:
            # decode requests past the knee: main requests first, then forks (hybrid_batch_time)
            ex_m = max(0.0, nd - n0)
            below = max(0.0, min(nf, n0 - nd)) if n0 != math.inf else nf
            ex_f = nf - below
            feats = [1.0, min(nd, n0) + ex_m, ex_m, pc, pc * pl]
            if with_forks:
                feats += [nf, ex_f]
            wgt = 1.0 / sec if relative else 1.0
            X.append([f * wgt for f in feats])
            y.append(sec * wgt)
        try:
            x = _lstsq(X, y)
        except CalibrationError:
            continue
        if with_forks:
            d0, g, ga, pf, pt, gf, gfa = x
        else:
            d0, g, ga, pf, pt = x
            gf, gfa = None, 0.0
        alpha = ga / g if g > 0 else 0.0
        try:
            params = CostModelParams(max(d0, 1e-12), max(g, 0.0), n0 if n0 != math.inf else 1e18, max(alpha, 0.0),
                                     max(pf, 0.0), max(pt, 0.0), None if gf is None else max(gf, 0.0))
        except ValueError:
            continue
        errs = [abs(hybrid_batch_time([(pl, pc)] if pc else (), nd, params, fork_count=nf) - sec) / sec
                for (pl, pc, nd, sec, nf) in rows]
        sse = sum(((hybrid_batch_time([(pl, pc)] if pc else (), nd, params, fork_count=nf) - sec) /
                   (sec if relative else 1.0)) ** 2 for (pl, pc, nd, sec, nf) in rows)
        if best is None or sse < best[0]:
            best = (sse, params, errs)
    if best is None:
        raise CalibrationError("no knee position gives a determined fit")
    _, params, errs = best
    report = {"max_rel_err": max(errs), "mean_rel_err": sum(errs) / len(errs), "rows": len(rows)}
    if max(errs) > max_rel_err:
        raise CalibrationError(f"calibrated T_h misses a table row by {max(errs):.1%} (> {max_rel_err:.0%})")
    return params, report


def load_table(path):
    """Rows of a profile CSV with header prefill_len,prefill_count,decode_count,seconds[,fork_count]."""
    import csv

    out = []
    with open(path) as f:
        for r in csv.DictReader(f):
            out.append((float(r["prefill_len"]), float(r["prefill_count"]), float(r["decode_count"]),
                        float(r["seconds"]), float(r.get("fork_count") or 0)))
    return out


def admitted_vs_load(params: CostModelParams, loads, k: int = 3, cand=None, n_a: int = 0):
    """|S| Algorithm 1 admits when every one of N main requests is a fresh candidate
    (equal priority inputs; the default SPEC.md:445 candidate), for each N in loads."""
    out = []
    for n in loads:
        q = [SpecCandidate(i, 1, float(i), **(cand or {})) for i in range(n)]
        r = select_step(q, (n, n, 0, n_a), params, SchedulerConfig(k=k, t_w=math.inf))
        out.append((n, len(r.selected), r.best))
    return out


__all__ = ["CostModelParams", "hybrid_batch_time", "decode_overhead", "prefill_overhead", "SpecCandidate",
           "expected_reduction", "GainBreakdown", "net_gain", "priority_key", "SchedulerConfig", "SelectResult",
           "select_step", "CalibrationError", "calibrate", "load_table", "admitted_vs_load"]
