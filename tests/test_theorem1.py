"""Theorem 1 (proof in App. A) on tiny LPs, as a pin of the oracle's
penalty solve (-m "not gpu").

For small VC and MIS instances the standard-form LP (Eq. 3 with the slack rows of App. C,
written out here from the graph, not taken from the oracle's encoding) is solved
exactly by scipy's HiGHS, which also returns a dual solution u*.  The same LP goes to
the oracle through its generic builder with x >= 0 only (no upper bound: Thm. 1 is
stated for Eq. 3), and the oracle's penalty solve with anchors (x_bar, u_bar) = (0, 0),
run to convergence, must satisfy
    ||A x(beta) - b|| <= (1 + sqrt 2) C* / beta   and   ||x(beta) - x*|| <= sqrt 6 C*,
C* = max(||x* - x_bar||, ||u* - u_bar||), for every beta tried; and with the anchors
set to the primal-dual pair itself (C* = 0) the penalty solution is that pair's x*.
"""
import numpy as np
import pytest

import oracle
from oracle import RefLP

scipy_opt = pytest.importorskip("scipy.optimize")

VC, MIS = 1, 2


def instance(seed, n=8, m=14):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    w = (1.0 + rng.integers(0, 9, n)).astype(np.float32)
    return n, src, dst, w


def standard_form(problem, n, rows, w):
    """Eq. 2 / App. B.2 rows with App. C slacks: row e = (u, v): x_u + x_v - s_e = 1 (VC)
    or x_u + x_v + s_e = 1 (MIS); z = (x, s) >= 0; cost c (VC) or -w (MIS, max as min)."""
    m = len(rows)
    A = np.zeros((m, n + m))
    for e, (u, v) in enumerate(rows):
        A[e, u] = A[e, v] = 1.0
        A[e, n + e] = -1.0 if problem == VC else 1.0
    c = np.concatenate([np.asarray(w, np.float64) * (1.0 if problem == VC else -1.0), np.zeros(m)])
    return A, np.ones(m), c


def oracle_lp(problem, n, rows, w):
    """the structural rows x_u + x_v >= 1 (VC) / <= 1 (MIS) as a generic LP, x in [0, inf)"""
    m = len(rows)
    cols = [[] for _ in range(n)]
    for e, (u, v) in enumerate(rows):
        cols[u].append(e)
        cols[v].append(e)
    colptr = np.concatenate([[0], np.cumsum([len(c) for c in cols])]).astype(np.int64)
    rowidx = np.array([e for c in cols for e in c], np.int32)
    sense = np.full(m, oracle.SENSE_GE if problem == VC else oracle.SENSE_LE, np.int8)
    return RefLP.generic(m, n, colptr, rowidx, np.ones(len(rowidx), np.float32), np.ones(m, np.float32),
                         np.asarray(w, np.float32), sense=sense, lo=np.zeros(n, np.float32),
                         hi=np.full(n, np.inf, np.float32), obj_sense=0 if problem == VC else 1)


def converged_point(lp, beta, A, b, epochs=4000, tol=1e-11):
    prev = None
    for _ in range(40):
        lp.solve(beta, epochs, mode=oracle.MODE_CYCLIC, seed=0, step_rule=oracle.STEP_LJ)
        z = lp.x()
        if prev is not None and np.max(np.abs(z - prev)) < tol:
            return z
        prev = z
    raise AssertionError("the penalty solve did not converge")


@pytest.mark.parametrize("problem", [VC, MIS])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_theorem1_bounds(problem, seed):
    n, src, dst, w = instance(seed)
    probe = RefLP.graph(problem, n, src, dst, vertex_w=w)
    eu, ev = probe.edges()
    rows = list(zip(eu.tolist(), ev.tolist()))
    A, b, c = standard_form(problem, n, rows, w)
    res = scipy_opt.linprog(c, A_eq=A, b_eq=b, bounds=[(0, None)] * A.shape[1], method="highs")
    assert res.status == 0
    zs, us = res.x, res.eqlin.marginals  # d(c^T z*)/db: the multiplier of -u^T (A z - b) in Eq. 5
    assert abs(c @ zs - b @ us) <= 1e-9 * max(1.0, abs(c @ zs))  # strong duality of the pair
    cstar = max(np.linalg.norm(zs), np.linalg.norm(us))  # anchors (0, 0)
    for beta in (0.5, 2.0, 8.0):
        lp = oracle_lp(problem, n, rows, w)
        z = converged_point(lp, beta, A, b)
        assert np.linalg.norm(A @ z - b) <= (1.0 + np.sqrt(2.0)) * cstar / beta + 1e-9
        assert np.linalg.norm(z - zs) <= np.sqrt(6.0) * cstar + 1e-9


@pytest.mark.parametrize("problem", [VC, MIS])
def test_anchors_at_a_primal_dual_pair_give_that_point(problem):
    # C* = 0: the bounds force x(beta) = x* and A x(beta) = b for every beta
    n, src, dst, w = instance(7)
    probe = RefLP.graph(problem, n, src, dst, vertex_w=w)
    rows = list(zip(*[a.tolist() for a in probe.edges()]))
    A, b, c = standard_form(problem, n, rows, w)
    res = scipy_opt.linprog(c, A_eq=A, b_eq=b, bounds=[(0, None)] * A.shape[1], method="highs")
    zs, us = res.x, res.eqlin.marginals
    for beta in (1.0, 5.0):
        lp = oracle_lp(problem, n, rows, w)
        lp.set_anchors(zbar=zs, ubar=us)
        z = converged_point(lp, beta, A, b)
        assert np.max(np.abs(z - zs)) <= 1e-6
        assert np.max(np.abs(A @ z - b)) <= 1e-6
