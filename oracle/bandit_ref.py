"""The Col-Bandit adaptive Top-K loop, restated on the CPU (test infrastructure only).

A deliberately plain full-ranking-per-iteration restatement of the reference
loop; it must agree with the reference reveal for reveal. Citations are to
/root/reference/pkg/src/colbandit:

* configuration defaults and validation — bandit.py:40-76, bounds.py:112-143;
* K checks and the K = 0 fast path — bandit.py:182-191;
* lazy warm-up after the first failed stop test, counted as an iteration —
  bandit.py:198-199, 285-296; ``init_one_per_row`` bandit.py:159-166;
  ``static_warmup`` bandit.py:139-156 with ``ceil_cells`` bandit.py:98-108;
* per-row state (hard bounds via math.fsum, estimate, radius, interval) —
  bandit.py:220-247 mirroring bounds.py:97-109, 146-158, 194-225, 259-263;
* ranking by (-proxy, i), i+ = argmin (lcb, i) over the Top-K, i- = argmax
  ucb over the rest with the lowest index on ties — bandit.py:249-284;
* row choice with the exhausted-row switch — bandit.py:301-312, 111-113;
* column choice: ``random() < eps`` always drawn, then ``integers(len(un))``
  or the first widest unrevealed column — bandit.py:314-326, 116-136;
* Welford update of the revealed row — oracle.py:305-314;
* result: Top-K of the final ranking, coverage = reveals / (N T) —
  bandit.py:349-350.

``run(..., indexed=True)`` keeps the ranking in the reference's own kind of
structures instead of re-sorting the pool every iteration — a sorted key list
of (-proxy, i) whose first K entries are the Top-K, a winner heap of (lcb, i)
and a loser heap of (-ucb, i) with lazy invalidation (bandit.py:249-284,
329-347) — so a 100k-row pool (cfg4) costs O(log N) per iteration like the
reference; both modes must produce the same result (tests/test_oracle_golden.py).

The RNG is numpy's ``default_rng(seed)`` exactly as the reference uses it.
Cells are supplied as the float64 N x T matrix the reference's oracle would
return from ``row_values`` (see maxsim_ref.cell_matrix).
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass

import numpy as np

EXPLORE_MODES = ("epsilon-greedy", "static-warmup", "uniform-row")
UNION_MODES = ("per-document", "per-document-and-size")


@dataclass(frozen=True)
class RefResult:
    topk: list
    coverage: float
    reveals: list
    iterations: int
    terminated_by: str


def ceil_cells(fraction: float, total: int) -> int:
    x = fraction * total
    nearest = round(x)
    if abs(x - nearest) < 1e-9 * max(1.0, total):
        return int(nearest)
    return math.ceil(x)


def log_term(n_rows: int, n_cols: int, delta: float, c: float, union_mode: str) -> float:
    arg = c * n_rows / delta
    if union_mode == "per-document-and-size":
        arg *= n_cols
    return max(math.log(arg), 0.0)


def fp_correction(n: int, n_cols: int) -> float:
    if 2 * n <= n_cols:
        return 1.0 - (n - 1) / n_cols
    return (1.0 - n / n_cols) * (1.0 + 1.0 / n)


def _pymin(a: float, b: float) -> float:
    return b if b < a else a


def _pymax(a: float, b: float) -> float:
    return b if b > a else a


def run(cells, lo, hi, k: int, *, delta: float = 0.01, alpha_ef: float = 1.0, epsilon: float = 0.1,
        explore_mode: str = "epsilon-greedy", gamma_init: float = 0.0, seed=0, c: float = 1.0,
        union_mode: str = "per-document", indexed: bool = False) -> RefResult:
    cells = np.asarray(cells, dtype=np.float64)
    n_rows, n_cols = cells.shape
    lo = np.broadcast_to(np.asarray(lo, dtype=np.float64), cells.shape)
    hi = np.broadcast_to(np.asarray(hi, dtype=np.float64), cells.shape)
    if k < 0:
        raise ValueError(f"k must be non-negative, got {k}")
    if explore_mode not in EXPLORE_MODES:
        raise ValueError(f"explore_mode must be one of {EXPLORE_MODES}, got {explore_mode!r}")
    if k > n_rows:
        raise ValueError(f"k={k} exceeds the number of documents ({n_rows})")
    if k == 0:
        return RefResult([], 0.0, [], 0, "separation")

    rng = np.random.default_rng(seed)
    warmed = k == n_rows or explore_mode == "uniform-row"
    eps = 1.0 if explore_mode == "uniform-row" else epsilon
    lt = log_term(n_rows, n_cols, delta, c, union_mode)
    T = n_cols
    lo_l = lo.tolist()
    hi_l = hi.tolist()
    revealed = [[False] * n_cols for _ in range(n_rows)]
    vals: list[list[float]] = [[] for _ in range(n_rows)]
    cnt = [0] * n_rows
    mean = [0.0] * n_rows
    m2 = [0.0] * n_rows
    proxy = np.zeros(n_rows)
    lcb = np.zeros(n_rows)
    ucb = np.zeros(n_rows)
    trace: list[tuple[int, int, float]] = []

    def refresh(i: int) -> None:
        n = cnt[i]
        obs = math.fsum(vals[i])
        un = [t for t in range(n_cols) if not revealed[i][t]]
        h_lo = obs + math.fsum(lo_l[i][t] for t in un)
        h_hi = obs + math.fsum(hi_l[i][t] for t in un)
        if n == 0:
            proxy[i], lcb[i], ucb[i] = 0.5 * (h_lo + h_hi), h_lo, h_hi
            return
        est = obs if n == T else T * (obs / n)
        proxy[i] = est
        if n <= 1:
            lcb[i], ucb[i] = h_lo, h_hi
            return
        sigma = math.sqrt(max(m2[i], 0.0) / (n - 1))
        r = alpha_ef * T * sigma * math.sqrt(2.0 * lt / n) * math.sqrt(fp_correction(n, T))
        lcb[i] = _pymin(_pymax(h_lo, est - r), h_hi)
        ucb[i] = _pymax(_pymin(h_hi, est + r), h_lo)

    def reveal(i: int, t: int) -> None:
        if revealed[i][t]:
            raise ValueError(f"cell ({i}, {t}) already revealed")
        v = float(cells[i, t])
        revealed[i][t] = True
        n = cnt[i] + 1
        cnt[i] = n
        d = v - mean[i]
        mean[i] += d / n
        m2[i] += d * (v - mean[i])
        vals[i].append(v)
        trace.append((i, t, v))

    for i in range(n_rows):
        refresh(i)
    idx = np.arange(n_rows)

    # ---- ranking structures of the indexed mode (bandit.py:249-284, 329-347)
    keys = None          # SortedList of (-proxy, i): the first k entries are the Top-K
    member = [False] * n_rows
    ver = [0] * n_rows   # bumped whenever a row's interval changes: older heap entries are stale
    win: list = []       # (lcb, i, ver) over members
    lose: list = []      # (-ucb, i, ver) over the rest
    key_of = [0.0] * n_rows

    def push(i: int) -> None:
        if member[i]:
            heapq.heappush(win, (float(lcb[i]), i, ver[i]))
        else:
            heapq.heappush(lose, (-float(ucb[i]), i, ver[i]))

    def rebuild() -> None:
        nonlocal keys
        from sortedcontainers import SortedList

        for i in range(n_rows):
            key_of[i] = -float(proxy[i]) + 0.0  # -0.0 ties with 0.0 (np.lexsort compares values)
        keys = SortedList((key_of[i], i) for i in range(n_rows))
        for i in range(n_rows):
            member[i] = False
        for _, i in keys[:k]:
            member[i] = True
        win.clear()
        lose.clear()
        for i in range(n_rows):
            ver[i] += 1
            push(i)

    def moved(i: int) -> None:
        """Row i was refreshed: re-rank it, swap Top-K membership across the boundary if it crossed."""
        keys.remove((key_of[i], i))
        key_of[i] = -float(proxy[i]) + 0.0
        keys.add((key_of[i], i))
        ver[i] += 1
        pos_in = keys.index((key_of[i], i)) < k
        if pos_in != member[i]:
            member[i] = pos_in
            # the row pushed across the boundary the other way: the new k-th entry, or the first of the rest
            j = keys[k - 1][1] if not pos_in else keys[k][1]
            member[j] = not pos_in
            push(j)
        push(i)

    def boundary():
        while True:
            l, i, v = win[0]
            if member[i] and v == ver[i]:
                i_plus = i
                break
            heapq.heappop(win)
        while lose:
            u, i, v = lose[0]
            if not member[i] and v == ver[i]:
                return i_plus, i, -u
            heapq.heappop(lose)
        return i_plus, -1, -math.inf

    if indexed:
        rebuild()
    iterations = 0
    terminated_by = "separation"
    order = None
    while True:
        iterations += 1
        if indexed:
            i_plus, i_minus, ucb_minus = boundary()
        else:
            order = np.lexsort((idx, -proxy))
            top, rest = order[:k], order[k:]
            i_plus = int(top[np.lexsort((top, lcb[top]))[0]])
            if len(rest):
                i_minus = int(rest[np.lexsort((rest, -ucb[rest]))[0]])
                ucb_minus = float(ucb[i_minus])
            else:
                i_minus, ucb_minus = -1, -math.inf
        if lcb[i_plus] >= ucb_minus:
            break
        if not warmed:
            warmed = True
            if explore_mode == "epsilon-greedy":
                for i in range(n_rows):
                    reveal(i, int(rng.integers(n_cols)))
            else:
                m = ceil_cells(gamma_init, n_rows * n_cols)
                if m:
                    for f in rng.choice(n_rows * n_cols, size=m, replace=False):
                        reveal(*divmod(int(f), n_cols))
            if trace:
                for i in range(n_rows):
                    refresh(i)
                if indexed:
                    rebuild()
            continue
        if len(trace) == n_rows * n_cols:
            terminated_by = "exhaustion"
            break
        w_plus = float(ucb[i_plus] - lcb[i_plus])
        w_minus = float(ucb[i_minus] - lcb[i_minus])
        i_star = i_plus if w_plus >= w_minus else i_minus
        un = [t for t in range(n_cols) if not revealed[i_star][t]]
        if not un:
            i_star = i_minus if i_star == i_plus else i_plus
            un = [t for t in range(n_cols) if not revealed[i_star][t]]
            if not un:
                raise RuntimeError("internal error: both boundary rows exhausted while unseparated")
        if rng.random() < eps:
            t_star = un[int(rng.integers(len(un)))]
        else:
            best, t_star = -math.inf, un[0]
            for t in un:
                w = hi_l[i_star][t] - lo_l[i_star][t]
                if w > best:
                    best, t_star = w, t
        reveal(i_star, t_star)
        refresh(i_star)
        if indexed:
            moved(i_star)
    topk = [int(i) for _, i in keys[:k]] if indexed else [int(i) for i in order[:k]]
    return RefResult(topk, len(trace) / (n_rows * n_cols), trace, iterations, terminated_by)


def full_rerank(cells, k: int) -> RefResult:
    """Reveal every cell row-major, rank by exactly rounded row sums — baselines.py:38-41, 89-97."""
    cells = np.asarray(cells, dtype=np.float64)
    n_rows, n_cols = cells.shape
    if not 0 <= k <= n_rows:
        raise ValueError(f"k must be in [0, {n_rows}], got {k}")
    trace = [(i, t, float(cells[i, t])) for i in range(n_rows) for t in range(n_cols)]
    sums = [math.fsum(cells[i].tolist()) for i in range(n_rows)]
    order = sorted(range(n_rows), key=lambda i: (-sums[i], i))
    return RefResult(order[:k], 1.0, trace, 0, "budget")
