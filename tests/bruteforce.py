"""Brute-force ground truth for tiny instances (independent of oracle/):
exhaustive enumeration over {0,1/2,1}^n (half-integral VC / edge-MIS LP
optima, Nemhauser-Trotter) and {0,1}^n (integer optima), and exhaustive
k-labellings for multiway cut."""
from __future__ import annotations

import itertools

import numpy as np


def unique_edges(n, src, dst):
    s = set()
    for u, v in zip(np.asarray(src).tolist(), np.asarray(dst).tolist()):
        if u != v:
            s.add((min(u, v), max(u, v)))
    return sorted(s)


def row_order(n, edges, hubs=True, hub_nnz=512):
    """R-17 written out: rows whose larger endpoint lies in a hub tile (32 consecutive
    vertex ids with more than hub_nnz incidences; VC / MIS only) in (u >> 14, v, u)
    order; then the other rows whose smaller endpoint lies in a hub tile, in
    (v >> 14, u, v) order; then the remaining rows, in (v, u) order."""
    tnz = {}
    for u, v in edges:
        tnz[u >> 5] = tnz.get(u >> 5, 0) + 1
        tnz[v >> 5] = tnz.get(v >> 5, 0) + 1

    def hub(x):
        return hubs and tnz[x >> 5] > hub_nnz

    first = [e for e in edges if hub(e[1])]
    mixed = [e for e in edges if not hub(e[1]) and hub(e[0])]
    rest = [e for e in edges if not hub(e[1]) and not hub(e[0])]
    return (sorted(first, key=lambda e: (e[0] >> 14, e[1], e[0])) + sorted(mixed, key=lambda e: (e[1] >> 14, e[0], e[1]))
            + sorted(rest, key=lambda e: (e[1], e[0])))


def incidence(n, rows):
    """per vertex: the rows where it is the larger endpoint, then the smaller (R-17)"""
    inc = [[] for _ in range(n)]
    for i, (u, v) in enumerate(rows):
        inc[v].append(i)
    for i, (u, v) in enumerate(rows):
        inc[u].append(i)
    return inc


def _grid_points(n, values):
    vals = np.array(values, dtype=np.float64)
    idx = np.indices((len(vals),) * n).reshape(n, -1).T
    return vals[idx]


def vc_lp_opt(n, edges, c):
    """min c.x s.t. x_u + x_v >= 1, x in [0,1]: optimum attained on {0,1/2,1}^n."""
    X = _grid_points(n, [0.0, 0.5, 1.0])
    ok = np.ones(len(X), bool)
    for u, v in edges:
        ok &= X[:, u] + X[:, v] >= 1.0
    return float((X[ok] @ np.asarray(c, np.float64)).min())


def vc_ip_opt(n, edges, c):
    X = _grid_points(n, [0.0, 1.0])
    ok = np.ones(len(X), bool)
    for u, v in edges:
        ok &= X[:, u] + X[:, v] >= 1.0
    return float((X[ok] @ np.asarray(c, np.float64)).min())


def mis_ip_opt(n, edges, w):
    X = _grid_points(n, [0.0, 1.0])
    ok = np.ones(len(X), bool)
    for u, v in edges:
        ok &= X[:, u] + X[:, v] <= 1.0
    return float((X[ok] @ np.asarray(w, np.float64)).max())


def mis_lp_opt(n, edges, w):
    X = _grid_points(n, [0.0, 0.5, 1.0])
    ok = np.ones(len(X), bool)
    for u, v in edges:
        ok &= X[:, u] + X[:, v] <= 1.0
    return float((X[ok] @ np.asarray(w, np.float64)).max())


def mwc_ip_opt(n, edges, ce, k, term_label):
    """min over labellings with terminals fixed of sum_e c_e [l_u != l_v]."""
    free = [v for v in range(n) if term_label[v] < 0]
    best = np.inf
    lab = np.array(term_label)
    for assign in itertools.product(range(k), repeat=len(free)):
        lab[free] = assign
        cost = sum(c for (u, v), c in zip(edges, ce) if lab[u] != lab[v])
        best = min(best, cost)
    return float(best)


def simplex_projection_bisect(y, iters=200):
    """Projection onto {x >= 0, sum x = 1} by bisection on tau in
    sum_l max(y_l - tau, 0) = 1 (a different algorithm from the sort-based one)."""
    y = np.asarray(y, np.float64)
    lo, hi = y.min() - 1.0, y.max()
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if np.maximum(y - mid, 0).sum() > 1.0:
            lo = mid
        else:
            hi = mid
    return np.maximum(y - 0.5 * (lo + hi), 0)
