"""Pins of the oracle against what the paper and the mathematics fix
(never against the oracle itself).  Every test names its pin.

P:L = /root/reference/PAPER.md line (not read at run time); S:L = SPEC.md line.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
from oracle import RefLP
from tests import bruteforce as bf

VC, MIS, MWC = 1, 2, 3


def dense_lp(A, b, c, sense=None, lo=None, hi=None, obj_sense=0, block_k=0, n_blocks=0, bits=64):
    A = np.asarray(A, np.float64)
    m, n = A.shape
    colptr = [0]
    rows, vals = [], []
    for j in range(n):
        nz = np.nonzero(A[:, j])[0]
        rows += nz.tolist()
        vals += A[nz, j].tolist()
        colptr.append(len(rows))
    return RefLP.generic(m, n, colptr, np.array(rows, np.int32), np.array(vals, np.float32), b, c,
                         sense=sense, lo=lo, hi=hi, obj_sense=obj_sense, block_k=block_k,
                         n_blocks=n_blocks, bits=bits)


def small_graph(n, m, seed):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    return src, dst


def regular_graph(name):
    if name == "K2":
        return 2, [(0, 1)], 1
    if name == "K3":
        return 3, [(0, 1), (0, 2), (1, 2)], 2
    if name == "C5":
        return 5, [(i, (i + 1) % 5) for i in range(5)], 2
    if name == "K4":
        return 4, [(a, b) for a in range(4) for b in range(a + 1, 4)], 3
    if name == "Q3":  # cube, 3-regular
        return 8, [(a, a ^ (1 << t)) for a in range(8) for t in range(3) if a < a ^ (1 << t)], 3
    if name == "K40":  # 39-regular: every tile of 32 vertices holds > 512 incidences (hub tiles)
        return 40, [(a, b) for a in range(40) for b in range(a + 1, 40)], 39
    if name == "Circ":  # circulant C_1024(1..12), 24-regular: all its tiles are hub tiles
        return 1024, [(a, (a + t) % 1024) for a in range(1024) for t in range(1, 13)], 24
    raise KeyError(name)


# ---------------------------------------------------------------------------
# Eq. 5 / Eq. 7 / Alg. 1 hand values (SPEC examples, re-derived by hand)
# ---------------------------------------------------------------------------
def test_objective_hand_value():
    # pin: S:105 — A=[1], b=1, c=1, beta=1, x=1 -> f = 1 + 0 + 0 + 1/2 = 1.5 (Eq. 5)
    lp = dense_lp([[1.0]], [1.0], [1.0])
    lp.set_x([1.0])
    assert lp.objective(1.0)["f_beta"] == pytest.approx(1.5, abs=1e-15)
    # pin: S:107 — same with ubar = 1: the -ubar^T(Ax-b) term vanishes at Ax = b
    lp.set_anchors(ubar=[1.0])
    assert lp.objective(1.0)["f_beta"] == pytest.approx(1.5, abs=1e-15)
    # pin: x = xbar and Ax = b -> f = c^T x for any ubar
    lp.set_anchors(zbar=[1.0], ubar=[3.0])
    assert lp.objective(1.0)["f_beta"] == pytest.approx(1.0, abs=1e-15)


def test_grad_hand_value():
    # pin: S:115 — A=[1], b=1, c=1, beta=2, x=0 -> 1 + 2*(0-1) + 0 = -1
    lp = dense_lp([[1.0]], [1.0], [1.0])
    assert lp.grad(2.0, 0) == pytest.approx(-1.0, abs=1e-15)


@pytest.mark.parametrize("A,beta,expect", [
    ([[1.0, 0.0], [0.0, 2.0]], 2.0, 2 * 4 + 0.5),   # columns (1,0),(0,2) -> 8.5
    ([[1.0, 0.0], [0.0, 1.0]], 1.0, 2.0),           # A = I, beta = 1 -> 2
])
def test_lmax_hand_value(A, beta, expect):
    # pin: Eq. 7 on EQ rows (no slack columns)
    lp = dense_lp(A, [1.0, 1.0], [1.0, 1.0])
    assert lp.solve(beta, 0)["L_max"] == pytest.approx(expect, abs=1e-15)


def test_lmax_counts_slack_columns():
    # pin: slack columns have ||a||^2 = 1, so L_max >= beta + 1/beta (Eq. 7 over [A | -I])
    lp = dense_lp([[0.5]], [1.0], [1.0], sense=[oracle.SENSE_GE])
    assert lp.solve(4.0, 0)["L_max"] == pytest.approx(4.0 * 1.0 + 0.25)


@pytest.mark.parametrize("bits", [64, 32])
def test_one_scd_step_hand_value(bits):
    # pin: S:166 — A=[1], b=1, c=1, beta=2, x=0: g=-1, L=2.5, x <- 0 + 1/2.5 = 0.4, r: -1 -> -0.6
    lp = dense_lp([[1.0]], [1.0], [1.0], bits=bits)
    assert lp.r()[0] == -1.0
    lp.step_unit(2.0, 0)
    assert lp.x()[0] == pytest.approx(0.4, rel=1e-6 if bits == 32 else 1e-15)
    assert lp.r()[0] == pytest.approx(-0.6, rel=1e-6 if bits == 32 else 1e-15)


def test_step_clamps_at_lower_bound():
    # pin: S:165 / Alg. 1 line 4 max(0, .) — x at 0 with positive gradient stays, r unchanged
    lp = dense_lp([[1.0]], [0.0], [5.0])
    r0 = lp.r().copy()
    lp.step_unit(1.0, 0)
    assert lp.x()[0] == 0.0 and np.array_equal(lp.r(), r0)


def test_step_clamps_at_upper_bound():
    # pin: box [lo, hi] (R-2): a strongly negative gradient stops at hi = 1
    lp = dense_lp([[1.0]], [10.0], [0.0])
    lp.step_unit(1.0, 0)  # g = 0 + 1*(0-10) = -10, L = 2: x = 5 -> clamp 1
    assert lp.x()[0] == 1.0
    assert lp.r()[0] == pytest.approx(-9.0)


# ---------------------------------------------------------------------------
# gradient = derivative of the objective (finite differences), all terms on
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(5))
def test_gradient_matches_finite_differences(seed):
    # pin: S:128 — every partial derivative matches the central difference of Eq. 5
    rng = np.random.default_rng(seed)
    m, n = 6, 9
    A = rng.normal(size=(m, n)) * (rng.random((m, n)) < 0.5)
    sense = rng.integers(0, 3, m).astype(np.int8)
    lp = dense_lp(A.astype(np.float32), rng.normal(size=m), rng.normal(size=n), sense=sense)
    N = lp.N
    z = rng.random(N)
    lp.set_x(z)
    lp.set_anchors(zbar=rng.normal(size=N), ubar=rng.normal(size=lp.m))
    beta, h = 3.0, 1e-6
    for j in range(N):
        zp, zm = z.copy(), z.copy()
        zp[j] += h
        zm[j] -= h
        lp.set_x(zp)
        fp = lp.objective(beta)["f_beta"]
        lp.set_x(zm)
        fm = lp.objective(beta)["f_beta"]
        lp.set_x(z)
        fd = (fp - fm) / (2 * h)
        assert lp.grad(beta, j) == pytest.approx(fd, rel=1e-6, abs=1e-6), j


# ---------------------------------------------------------------------------
# monotone decrease per exact coordinate step (BASELINE north star)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("rule", [oracle.STEP_LMAX, oracle.STEP_LJ])
@pytest.mark.parametrize("problem", [VC, MIS])
def test_penalty_never_increases_per_step_graph(problem, rule):
    src, dst = small_graph(12, 30, 7 + problem)
    w = np.random.default_rng(1).uniform(1, 10, 12).astype(np.float32)
    lp = RefLP.graph(problem, 12, src, dst, vertex_w=w)
    beta = 10.0
    f = lp.objective(beta)["f_beta"]
    rng = np.random.default_rng(3)
    for _ in range(600):
        lp.step_unit(beta, int(rng.integers(lp.U)), rule)
        f2 = lp.objective(beta)["f_beta"]
        assert f2 <= f + 1e-12 * max(1.0, abs(f))
        f = f2


@pytest.mark.parametrize("rule", [oracle.STEP_LMAX, oracle.STEP_LJ])
def test_penalty_never_increases_per_block_step_mwc(rule):
    # block steps with simplex projection are also descent steps (projected gradient on a
    # block whose curvature is <= L): App. E
    side = 3
    src = [r * side + c for r in range(side) for c in range(side - 1)] + \
          [r * side + c for r in range(side - 1) for c in range(side)]
    dst = [s + 1 for s in src[: side * (side - 1)]] + [s + side for s in src[side * (side - 1):]]
    ew = np.random.default_rng(2).exponential(1.0, len(src)).astype(np.float32)
    lp = RefLP.graph(MWC, 9, src, dst, edge_w=ew, k=3, terminals=[0, 2, 8], t_per_label=1)
    beta = 10.0
    f = lp.objective(beta)["f_beta"]
    rng = np.random.default_rng(5)
    for _ in range(500):
        lp.step_unit(beta, int(rng.integers(lp.U)), rule)
        f2 = lp.objective(beta)["f_beta"]
        assert f2 <= f + 1e-12 * max(1.0, abs(f))
        f = f2
    x = lp.x()
    for v in range(9):  # App. C.3: blocks stay on the simplex
        blk = x[v * 3: v * 3 + 3]
        assert blk.min() >= 0 and abs(blk.sum() - 1) < 1e-12


# ---------------------------------------------------------------------------
# closed-form x(beta) (KKT of Eq. 5) on d-regular vertex-transitive graphs
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["K2", "K3", "C5", "K4", "Q3"])
@pytest.mark.parametrize("mode", [oracle.MODE_DET, oracle.MODE_ASYNC, oracle.MODE_CYCLIC])
def test_vc_converges_to_closed_form(name, mode):
    # unit costs, ubar = xbar = 0: slacks 0 and x_v = beta(d beta - 1)/(2 d beta^2 + 1)
    n, edges, d = regular_graph(name)
    beta = 10.0
    src = [u for u, _ in edges]
    dst = [v for _, v in edges]
    lp = RefLP.graph(VC, n, src, dst, vertex_w=np.ones(n, np.float32))
    lp.solve(beta, 4000, mode=mode, seed=11, step_rule=oracle.STEP_LJ)
    x = lp.x()
    expect = beta * (d * beta - 1) / (2 * d * beta * beta + 1)
    np.testing.assert_allclose(x[:n], expect, atol=1e-9)
    np.testing.assert_allclose(x[n:], 0.0, atol=1e-9)
    if name == "K3":
        assert expect == pytest.approx(0.473815, abs=1e-6)


@pytest.mark.parametrize("name", ["K3", "Q3", "K40", "Circ"])
@pytest.mark.parametrize("mode", [oracle.MODE_PI_TILE_SYNC, oracle.MODE_HUBLAG_REPLAY])
@pytest.mark.parametrize("problem", [VC, MIS])
def test_replays_converge_to_closed_form(problem, mode, name):
    # the two replays of the GPU schedules (mode 4: THETIS_MODE_ASYNC's tile-synchronous
    # sweep; mode 3: the hub-lag schedule, R-22, with hub tiles on K40 / Circ) are other
    # ways to minimise the same strongly convex f_beta: both reach Eq. 5's unique minimiser
    # x(beta), the same closed forms as Alg. 1 (VC beta(d beta - 1)/(2 d beta^2 + 1), MIS
    # beta(d beta + 1)/(2 d beta^2 + 1)), slacks 0
    # (beta = 2 on the dense graphs: the same closed form, reached in fewer epochs)
    n, edges, d = regular_graph(name)
    beta = 2.0 if d > 3 else 10.0
    lp = RefLP.graph(problem, n, [u for u, _ in edges], [v for _, v in edges], vertex_w=np.ones(n, np.float32))
    lp.solve(beta, 5000, mode=mode, seed=13, step_rule=oracle.STEP_LMAX)
    expect = beta * (d * beta + (1 if problem == MIS else -1)) / (2 * d * beta * beta + 1)
    np.testing.assert_allclose(lp.x()[:n], expect, atol=1e-7)
    np.testing.assert_allclose(lp.x()[n:], 0.0, atol=1e-7)
    assert lp.objective(beta)["drift_inf"] < 1e-10


@pytest.mark.parametrize("problem", [VC, MIS, MWC])
def test_pi_tile_sync_replay_is_monotone(problem):
    # mode 4 under 1/L_max is a descent method epoch by epoch: a structural tile's columns
    # step together from one state, and with two structural entries per row the tile's
    # Hessian block has lambda_max <= 2 beta max_j ||a_j||^2 + 1/beta < 2 L_max (Eq. 7), so
    # the synchronous step with 1/L_max decreases f_beta; slack tiles and MWC edge-label
    # tiles touch disjoint rows (a diagonal block); k-blocks step one at a time
    if problem == MWC:
        side = 12
        src = [r * side + c for r in range(side) for c in range(side - 1)] + \
              [r * side + c for r in range(side - 1) for c in range(side)]
        dst = [s + 1 for s in src[: side * (side - 1)]] + [s + side for s in src[side * (side - 1):]]
        ew = np.random.default_rng(2).exponential(1.0, len(src)).astype(np.float32)
        lp = RefLP.graph(MWC, side * side, src, dst, edge_w=ew, k=3, terminals=[0, 11, 143], t_per_label=1)
    else:
        src, dst = small_graph(300, 2400, 5)
        w = np.random.default_rng(4).uniform(1, 10, 300).astype(np.float32)
        lp = RefLP.graph(problem, 300, src, dst, vertex_w=w)
    beta = 10.0
    f = lp.objective(beta)["f_beta"]
    for e in range(40):
        lp.solve(beta, 1, mode=oracle.MODE_PI_TILE_SYNC, seed=100 + e, step_rule=oracle.STEP_LMAX)
        f2 = lp.objective(beta)["f_beta"]
        assert f2 <= f + 1e-12 * max(1.0, abs(f))
        f = f2


def test_pi_tile_sync_equals_alg1_when_tiles_are_independent():
    # with n a multiple of 32 and every edge joining two different tiles, no two units of a
    # tile share a row: the tile-synchronous sweep (mode 4) and Alg. 1 one unit at a time
    # (mode 1) perform the same operations on the same values -- bit-identical
    n = 256
    rng = np.random.default_rng(8)
    u = rng.integers(0, n, 3000)
    v = (u + 32 * rng.integers(1, n // 32, 3000)) % n
    w = rng.uniform(1, 10, n).astype(np.float32)
    for problem in (VC, MIS):
        for rule in (oracle.STEP_LMAX, oracle.STEP_LJ):
            a = RefLP.graph(problem, n, u.astype(np.int32), v.astype(np.int32), vertex_w=w)
            b = RefLP.graph(problem, n, u.astype(np.int32), v.astype(np.int32), vertex_w=w)
            a.solve(10.0, 7, mode=oracle.MODE_ASYNC, seed=21, step_rule=rule)
            b.solve(10.0, 7, mode=oracle.MODE_PI_TILE_SYNC, seed=21, step_rule=rule)
            assert np.array_equal(a.x(), b.x()) and np.array_equal(a.r(), b.r())


def test_hublag_replay_differs_from_alg1_but_not_at_the_fixed_point():
    # mode 3 is a different schedule (slacks first, hubs one synchronous lagged step): after
    # a few epochs on a hub graph it is measurably off Alg. 1's trajectory, after many both
    # sit at the same x(beta) (the distances DESIGN.md R-22 reports at scale)
    n, edges, d = regular_graph("K40")
    src, dst = [e[0] for e in edges], [e[1] for e in edges]
    w = np.random.default_rng(3).uniform(1, 10, n).astype(np.float32)
    lag = RefLP.graph(VC, n, src, dst, vertex_w=w)
    alg1 = RefLP.graph(VC, n, src, dst, vertex_w=w)
    lag.solve(2.0, 5, mode=oracle.MODE_HUBLAG_REPLAY, seed=4)
    alg1.solve(2.0, 5, mode=oracle.MODE_ASYNC, seed=4)
    assert np.abs(lag.x() - alg1.x()).max() > 1e-4
    lag.solve(2.0, 3000, mode=oracle.MODE_HUBLAG_REPLAY, seed=5)
    alg1.solve(2.0, 3000, mode=oracle.MODE_ASYNC, seed=5)
    assert np.abs(lag.x() - alg1.x()).max() < 1e-9


@pytest.mark.parametrize("name", ["K2", "K3", "C5", "Q3"])
def test_mis_converges_to_closed_form(name):
    # MAX w^T x with LE rows: x_v = beta(d beta + 1)/(2 d beta^2 + 1); K2: 0.547264 (beta = 10)
    n, edges, d = regular_graph(name)
    beta = 10.0
    lp = RefLP.graph(MIS, n, [u for u, _ in edges], [v for _, v in edges],
                     vertex_w=np.ones(n, np.float32))
    lp.solve(beta, 4000, mode=oracle.MODE_DET, seed=3, step_rule=oracle.STEP_LMAX)
    expect = beta * (d * beta + 1) / (2 * d * beta * beta + 1)
    np.testing.assert_allclose(lp.x()[:n], expect, atol=1e-9)
    if name == "K2":
        assert expect == pytest.approx(0.547264, abs=1e-6)
        # App. C.2: alpha = 2x - 1 and x/(1+alpha) = (1/2, 1/2) exactly
        sel, res = lp.round(oracle.ROUND_MIS_GREEDY)
        assert res["eps_or_alpha"] == pytest.approx(2 * expect - 1, abs=1e-6)


def test_lp_value_approaches_bruteforce_optimum_as_beta_grows():
    # Thm. 1: |c^T x(beta) - c^T x*| = O(1/beta); LP* by brute force over {0,1/2,1}^n
    src, dst = small_graph(9, 20, 4)
    w = np.random.default_rng(9).uniform(1, 10, 9).astype(np.float32)
    edges = bf.unique_edges(9, src, dst)
    lp_star = bf.vc_lp_opt(9, edges, w)
    gaps, epss = [], []
    for beta in (10.0, 100.0, 1000.0):
        lp = RefLP.graph(VC, 9, src, dst, vertex_w=w)
        lp.solve(beta, 20000, mode=oracle.MODE_CYCLIC, step_rule=oracle.STEP_LJ)
        o = lp.objective(beta)
        assert o["lp_obj"] < lp_star  # the penalty trades feasibility for cost
        gaps.append(lp_star - o["lp_obj"])
        epss.append(o["max_violation_eps"])
    # both the objective gap and the infeasibility shrink like 1/beta
    for a, b in ((gaps[0], gaps[1]), (gaps[1], gaps[2]), (epss[0], epss[1]), (epss[1], epss[2])):
        assert 8.0 < a / b < 12.0


# ---------------------------------------------------------------------------
# residual maintenance, encodings
# ---------------------------------------------------------------------------
def test_maintained_residual_equals_recomputed():
    src, dst = small_graph(40, 150, 2)
    w = np.random.default_rng(0).uniform(1, 10, 40).astype(np.float32)
    for problem in (VC, MIS):
        lp = RefLP.graph(problem, 40, src, dst, vertex_w=w)
        lp.solve(10.0, 30, mode=oracle.MODE_ASYNC, seed=5)
        assert lp.objective(10.0)["drift_inf"] < 1e-12


def hub_graph(n, m, seed):
    # random edges over four 2^14 ranges plus two hub tiles (ids 0-31 and 20000-20031)
    # with > 512 incidences each
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    hs = np.concatenate([rng.integers(0, 32, 700), rng.integers(20000, 20032, 700)])
    hd = rng.integers(0, n, 1400)
    return (np.concatenate([src, hs]).astype(np.int32), np.concatenate([dst, hd]).astype(np.int32))


@pytest.mark.parametrize("problem", [VC, MIS, MWC])
def test_graph_row_order_and_incidence(problem):
    # R-17: hub-partitioned row order; every column lists its max-endpoint rows, then its
    # min-endpoint rows, each ascending (checked against the plain definition)
    n = 4 << 14
    src, dst = hub_graph(n, 3000, 21)
    edges = bf.unique_edges(n, src, dst)
    if problem == MWC:
        lp = RefLP.graph(MWC, n, src, dst, edge_w=np.ones(len(src), np.float32), k=2,
                         terminals=[1, 2], t_per_label=1)
    else:
        lp = RefLP.graph(problem, n, src, dst, vertex_w=np.ones(n, np.float32))
    eu, ev = lp.edges()
    want = bf.row_order(n, edges, hubs=problem != MWC)
    if problem != MWC:
        assert want != sorted(edges, key=lambda e: (e[1], e[0]))  # the hub part is non-empty
        assert want != sorted(edges, key=lambda e: (e[0] >> 14, e[1], e[0]))
        # three parts: hub max endpoint; hub min endpoint only (ranged by the max endpoint);
        # the rest
        hub = lambda x: x < 32 or 20000 <= x < 20032  # noqa: E731
        part = [0 if hub(e[1]) else 1 if hub(e[0]) else 2 for e in want]
        assert part == sorted(part) and set(part) == {0, 1, 2}
        mixed = [e for e, p in zip(want, part) if p == 1]
        assert mixed == sorted(mixed, key=lambda e: (e[1] >> 14, e[0], e[1])) != sorted(mixed, key=lambda e: (e[1], e[0]))
    assert list(zip(eu.tolist(), ev.tolist())) == want
    if problem != MWC:
        colptr, rowidx, _ = lp.csc()
        inc = bf.incidence(n, want)
        for v in list(range(0, 64)) + list(range(19990, 20040)) + list(range(0, n, 97)):
            assert rowidx[colptr[v]:colptr[v + 1]].tolist() == inc[v]


def test_graph_encoding_counts():
    # VC/MIS: one row per unique undirected non-loop edge, 2 structural nnz + 1 slack per row
    # (Fig. 3 NNZ:PV ~ 3:1); MWC: 2km rows, 6km structural nnz, 2km slacks
    src, dst = small_graph(30, 200, 8)
    edges = bf.unique_edges(30, src, dst)
    w = np.ones(30, np.float32)
    lp = RefLP.graph(VC, 30, src, dst, vertex_w=w)
    assert lp.m == len(edges) and lp.nnz_struct == 2 * len(edges) and lp.n_ineq == len(edges)
    eu, ev = lp.edges()
    assert list(zip(eu.tolist(), ev.tolist())) == bf.row_order(30, edges)
    b, sense, c = lp.rows()
    assert (b == 1).all() and (sense == oracle.SENSE_GE).all()
    lpm = RefLP.graph(MIS, 30, src, dst, vertex_w=w)
    b, sense, c = lpm.rows()
    assert (sense == oracle.SENSE_LE).all() and (c == -1).all()
    k = 4
    lpc = RefLP.graph(MWC, 30, src, dst, edge_w=np.ones(len(src), np.float32), k=k,
                      terminals=[0, 1, 2, 3], t_per_label=1)
    me = len(edges)
    assert lpc.m == 2 * k * me and lpc.nnz_struct == 6 * k * me and lpc.n_ineq == 2 * k * me
    assert lpc.n_struct == 30 * k + me * k and lpc.U == 30 + me * k + 2 * k * me


def test_fig3_size_ratios(golden_dir=None):
    # pin: tests/golden/fig3_sizes.txt (PAPER Fig. 3): NNZ/PV ~ 3 for VC and MIS,
    # matching one row per edge with 2 vertex nonzeros + 1 slack; MC NNZ ~ 8km + kn with
    # PV ~ 2km + n (Google+, n = 211186 printed at P:1566-1567, k = 3 at P:609)
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "fig3_sizes.txt")
    rows = [ln.split() for ln in open(path) if ln.strip() and not ln.startswith("#")]
    for inst, prob, pv, nnz in rows:
        pv, nnz = float(pv), float(nnz)
        if prob in ("VC", "MIS"):
            assert 2.9 <= nnz / pv <= 3.2, inst
    gp = [r for r in rows if r[0] == "Google+" and r[1] == "MC"][0]
    n, k = 211186, 3
    m = (float(gp[2]) * 1e6 - n) / (2 * k)
    assert abs(8 * k * m + k * n - float(gp[3]) * 1e6) / (float(gp[3]) * 1e6) < 0.01


def test_generic_builder_rejects_bad_input():
    with pytest.raises(oracle.OracleError):
        RefLP.generic(1, 1, [0, 1], [3], None, [1.0], [1.0])  # row out of range
    with pytest.raises(oracle.OracleError):
        RefLP.generic(1, 1, [0, 1], [0], None, [1.0], [1.0], lo=[1.0], hi=[0.0])  # lo > hi
    with pytest.raises(oracle.OracleError):
        RefLP.graph(VC, 3, [0], [5], vertex_w=np.ones(3, np.float32))  # vertex out of range


# ---------------------------------------------------------------------------
# simplex projection (App. E)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("y,expect", [
    ([0.5, 0.5, 0.5], [1 / 3, 1 / 3, 1 / 3]),
    ([2.0, 0.0, 0.0], [1.0, 0.0, 0.0]),
    ([0.7, 0.2, 0.0], [0.7 + 0.1 / 3, 0.2 + 0.1 / 3, 0.1 / 3]),
])
def test_simplex_projection_examples(y, expect):
    np.testing.assert_allclose(oracle.project_simplex(y), expect, atol=1e-15)


def test_simplex_projection_against_bisection():
    rng = np.random.default_rng(0)
    for _ in range(300):
        k = int(rng.integers(2, 9))
        y = rng.normal(size=k) * rng.choice([0.1, 1.0, 5.0])
        np.testing.assert_allclose(oracle.project_simplex(y), bf.simplex_projection_bisect(y),
                                   atol=1e-12)


# ---------------------------------------------------------------------------
# sweep orders
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n_tiles", [1, 2, 3, 4, 5, 7, 8, 9, 31, 32, 33, 1000, 4096, 4097, 65537])
def test_tile_permutation_is_bijection(n_tiles):
    for e in range(3):
        p = oracle.tile_perm(n_tiles, 1234, e)
        assert sorted(p.tolist()) == list(range(n_tiles))
    if n_tiles > 8:
        assert not np.array_equal(oracle.tile_perm(n_tiles, 1234, 0), oracle.tile_perm(n_tiles, 1234, 1))


def _unit_rows(lp):
    """rows touched by each structural unit (from the exported CSC)"""
    cp, ri, _ = lp.csc()
    k = max(lp.block_k, 1)
    rows = []
    for u in range(lp.n_blocks + (lp.n_struct - lp.n_blocks * lp.block_k)):
        if u < lp.n_blocks:
            cols = range(u * k, u * k + k)
        else:
            cols = [lp.n_blocks * lp.block_k + (u - lp.n_blocks)]
        rows.append(set(ri[cp[j]:cp[j + 1]].tolist() for j in cols for _ in [0]) if False else
                    set(int(i) for j in cols for i in ri[cp[j]:cp[j + 1]]))
    return rows


def _fmix32(h):
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & 0xFFFFFFFF
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & 0xFFFFFFFF
    h ^= h >> 16
    return h


@pytest.mark.parametrize("problem", [VC, MWC])
def test_colouring_is_proper_and_first_fit(problem):
    # definition (R-5): proper (no two units of a class share a row) and first-fit in
    # priority order (largest degree first): colour(u) = mex of the colours of the
    # higher-priority conflicting units
    src, dst = small_graph(40, 120, 12)
    if problem == VC:
        lp = RefLP.graph(VC, 40, src, dst, vertex_w=np.ones(40, np.float32))
    else:
        lp = RefLP.graph(MWC, 40, src, dst, edge_w=np.ones(120, np.float32), k=3,
                         terminals=[0, 1, 2], t_per_label=1)
    seed = 0xABCDEF0123
    K, col = lp.colouring(seed)
    rows = _unit_rows(lp)
    S = len(rows)
    key = _fmix32(seed & 0xFFFFFFFF) ^ (seed >> 32)
    cp, _, _ = lp.csc()
    k = max(lp.block_k, 1)

    def deg(u):
        cols = range(u * k, u * k + k) if u < lp.n_blocks else [lp.n_blocks * lp.block_k + u - lp.n_blocks]
        return sum(int(cp[j + 1] - cp[j]) for j in cols)

    # priority: largest degree first, then the larger hash, then the smaller id
    prio = [(deg(u), _fmix32(u ^ key)) for u in range(S)]
    assert (col[S:] == K).all()
    for u in range(S):
        if col[u] < 0:
            continue
        nb = [w for w in range(S) if w != u and col[w] >= 0 and rows[u] & rows[w]]
        assert all(col[w] != col[u] for w in nb)
        higher = {int(col[w]) for w in nb if (prio[w], -w) > (prio[u], -u)}
        assert col[u] not in higher and all(c in higher for c in range(col[u]))


# ---------------------------------------------------------------------------
# rounding
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(8))
def test_vc_rounding_bounds_against_bruteforce(seed):
    # P:139-146 (threshold 1/2 costs <= 2x fractional), Lemma 1: cost <= 2 c^T x/(1-eps);
    # feasible; IP* <= cost; and after a long solve cost <= 2 IP* (BASELINE north star)
    n = 10 + seed % 4
    src, dst = small_graph(n, 3 * n, 100 + seed)
    w = np.random.default_rng(seed).uniform(1, 10, n).astype(np.float32)
    edges = bf.unique_edges(n, src, dst)
    ip = bf.vc_ip_opt(n, edges, w)
    lp_star = bf.vc_lp_opt(n, edges, w)
    assert lp_star <= ip <= 2 * lp_star + 1e-9
    lp = RefLP.graph(VC, n, src, dst, vertex_w=w)
    lp.solve(10.0, 3000, mode=oracle.MODE_DET, seed=seed, step_rule=oracle.STEP_LJ)
    x = lp.x()[:n].astype(np.float32)
    for rule in (oracle.ROUND_VC_HALF, oracle.ROUND_VC_FIXUP):
        sel, res = lp.round_x(x, rule)
        assert res["feasible"] == 1
        assert all(sel[u] or sel[v] for u, v in edges)
        assert res["cost"] >= ip - 1e-9
        assert res["cost"] == pytest.approx(float(w[sel == 1].astype(np.float64).sum()))
    sel, res = lp.round_x(x, oracle.ROUND_VC_HALF)
    eps = res["eps_or_alpha"]
    assert eps < 1 and res["cost"] <= 2 * float(w.astype(np.float64) @ x) / (1 - eps) + 1e-6
    assert res["cost"] <= 2 * ip + 1e-9
    # the repaired point Pi(x/(1-eps)) is feasible (Lemma 1) and so costs >= LP*
    xt = np.minimum(x.astype(np.float64) / (1 - eps), 1.0)
    assert all(xt[u] + xt[v] >= 1 - 1e-6 for u, v in edges)
    assert float(w.astype(np.float64) @ xt) >= lp_star - 1e-4


@pytest.mark.parametrize("n", [3, 4, 6])
def test_vc_rounding_complete_graph_symmetric_point(n):
    # K_n, unit costs, symmetric fixed point x_v = beta(d beta-1)/(2 d beta^2+1) < 1/2:
    # VC_HALF (tau = (1-eps)/2 = x exactly) selects all n <= 2(n-1);
    # VC_FIXUP selects {0..n-2} (ties to the smaller id): n-1 = IP*
    edges = [(a, b) for a in range(n) for b in range(a + 1, n)]
    lp = RefLP.graph(VC, n, [a for a, _ in edges], [b for _, b in edges], vertex_w=np.ones(n, np.float32))
    d, beta = n - 1, 10.0
    x = np.full(n, np.float32(beta * (d * beta - 1) / (2 * d * beta * beta + 1)), np.float32)
    sel, res = lp.round_x(x, oracle.ROUND_VC_HALF)
    assert sel.sum() == n and res["fallback"] == 0
    sel, res = lp.round_x(x, oracle.ROUND_VC_FIXUP)
    assert sel.tolist() == [1] * (n - 1) + [0] and res["cost"] == n - 1


def test_vc_rounding_fallback_when_eps_ge_1():
    # Lemma 1 needs eps in [0, 1): at x = 0 eps = 1 -> threshold 1/2 + fix-up, fallback flagged
    lp = RefLP.graph(VC, 4, [0, 1, 2], [1, 2, 3], vertex_w=np.array([1, 2, 3, 4], np.float32))
    sel, res = lp.round_x(np.zeros(4, np.float32), oracle.ROUND_VC_HALF)
    assert res["fallback"] == 1 and res["feasible"] == 1
    assert sel.tolist() == [1, 1, 1, 0]  # x ties -> smaller cost per edge


@pytest.mark.parametrize("seed", range(6))
def test_mis_rounding_against_bruteforce(seed):
    # greedy repair: independent and maximal; weight <= IP*; contains {x~ > 1/2} when x~
    # is feasible; the packing repair x~ = x/(1+alpha) is feasible (App. C.2)
    n = 10 + seed % 5
    src, dst = small_graph(n, 2 * n, 200 + seed)
    w = np.random.default_rng(seed).uniform(1, 10, n).astype(np.float32)
    edges = bf.unique_edges(n, src, dst)
    ip = bf.mis_ip_opt(n, edges, w)
    lp = RefLP.graph(MIS, n, src, dst, vertex_w=w)
    lp.solve(10.0, 3000, mode=oracle.MODE_DET, seed=seed, step_rule=oracle.STEP_LJ)
    x = lp.x()[:n].astype(np.float32)
    sel, res = lp.round_x(x, oracle.ROUND_MIS_GREEDY)
    assert res["feasible"] == 1
    assert all(not (sel[u] and sel[v]) for u, v in edges)
    adj = {v: set() for v in range(n)}
    for u, v in edges:
        adj[u].add(v)
        adj[v].add(u)
    assert all(sel[v] or any(sel[u] for u in adj[v]) for v in range(n))  # maximal
    assert res["cost"] <= ip + 1e-9
    alpha = res["eps_or_alpha"]
    xt = x.astype(np.float64) / (1 + alpha)
    assert all(xt[u] + xt[v] <= 1 + 1e-6 for u, v in edges)
    for v in range(n):
        if xt[v] > 0.5 + 1e-6:
            assert sel[v] == 1


def test_mwc_path_costs_one_for_every_rep():
    # path s - v - t, k = 2, x_v = (1/2, 1/2): every (theta, sigma) cuts exactly one edge
    lp = RefLP.graph(MWC, 3, [0, 1], [1, 2], edge_w=np.ones(2, np.float32), k=2,
                     terminals=[0, 2], t_per_label=1)
    x = np.zeros(lp.n_struct, np.float32)
    x[0:2] = [1, 0]
    x[2:4] = [0.5, 0.5]
    x[4:6] = [0, 1]
    for seed in range(20):
        lab, res = lp.round_x(x, oracle.ROUND_MWC_CKR, seed=seed, reps=1)
        assert res["cost"] == 1.0 and lab[0] == 0 and lab[2] == 1


def test_mwc_path_lp_value():
    # path s - v - t with k = 2: LP = IP = 1; the solve approaches it
    lp = RefLP.graph(MWC, 3, [0, 1], [1, 2], edge_w=np.ones(2, np.float32), k=2,
                     terminals=[0, 2], t_per_label=1)
    lp.solve(1000.0, 20000, mode=oracle.MODE_CYCLIC, step_rule=oracle.STEP_LJ)
    assert lp.objective(1000.0)["lp_obj"] == pytest.approx(1.0, abs=5e-3)


@pytest.mark.parametrize("seed", range(3))
def test_mwc_rounding_against_bruteforce(seed):
    # 3x3 grid, k = 3: terminals keep their labels; cost >= IP* (3^6 labellings);
    # best-of-reps never worse than any single rep
    side, k = 3, 3
    src = [r * side + c for r in range(side) for c in range(side - 1)] + \
          [r * side + c for r in range(side - 1) for c in range(side)]
    dst = [s + 1 for s in src[: side * (side - 1)]] + [s + side for s in src[side * (side - 1):]]
    ew = np.random.default_rng(seed).exponential(1.0, len(src)).astype(np.float32)
    terms = [0, 2, 8]
    lp = RefLP.graph(MWC, 9, src, dst, edge_w=ew, k=k, terminals=terms, t_per_label=1)
    lp.solve(10.0, 2000, mode=oracle.MODE_DET, seed=seed, step_rule=oracle.STEP_LJ)
    eu, ev = lp.edges()
    tl = [-1] * 9
    for l, v in enumerate(terms):
        tl[v] = l
    order = {(min(a, b), max(a, b)): i for i, (a, b) in enumerate(zip(src, dst))}
    ce = [float(ew[order[(int(u), int(v))]]) for u, v in zip(eu, ev)]
    ip = bf.mwc_ip_opt(9, list(zip(eu.tolist(), ev.tolist())), ce, k, tl)
    lab, res = lp.round(oracle.ROUND_MWC_CKR, seed=seed, reps=10)
    assert [lab[v] for v in terms] == [0, 1, 2]
    assert res["cost"] >= ip - 1e-9
    singles = [lp.round(oracle.ROUND_MWC_CKR, seed=seed, reps=t + 1)[1]["cost"] for t in range(10)]
    assert res["cost"] == min(singles)


def test_mwc_round_precondition():
    lp = RefLP.graph(MWC, 3, [0, 1], [1, 2], edge_w=np.ones(2, np.float32), k=2,
                     terminals=[0, 2], t_per_label=1)
    x = np.zeros(lp.n_struct, np.float32)
    x[2:4] = [0.9, 0.9]
    with pytest.raises(oracle.OracleError) as e:
        lp.round_x(x, oracle.ROUND_MWC_CKR)
    assert e.value.code == -6


def test_fp32_build_tracks_fp64_build():
    # the fp32 build is the same plain arithmetic; on config-1-like input it stays within
    # 1e-6 of fp64 after 20 epochs (R-7: fp32 state is what BASELINE fixes)
    import inputs
    g = inputs.make_graph(inputs.CONFIGS["vc_er_1k"])
    a = RefLP.graph(VC, g.n, g.src, g.dst, vertex_w=g.vertex_w, bits=64)
    b = RefLP.graph(VC, g.n, g.src, g.dst, vertex_w=g.vertex_w, bits=32)
    for lp in (a, b):
        lp.solve(10.0, 20, mode=oracle.MODE_DET, seed=71)
    assert np.abs(a.x() - b.x()).max() < 1e-6
    assert np.abs(a.r() - b.r()).max() < 1e-6


def test_column_dot_is_the_contracts_tree():
    # R-7: lanes at CSC positions 0, 1, 2 combine by halving, off = 2 first:
    # p0 = (r0 + r2) + r1.  With r = (1e8, 1, -1e8) in fp32 that is (1e8 - 1e8) + 1 = 1,
    # while the plain sequential sum (1e8 + 1) - 1e8 rounds to 0 (fp32 spacing at 1e8 is 8).
    # One EQ row per entry, b = -r, z = 0, c = 0, beta = 1: the gradient is the dot itself.
    b = np.array([-1e8, -1.0, 1e8], np.float32)
    lp = RefLP.generic(3, 1, np.array([0, 3]), np.array([0, 1, 2], np.int32), np.ones(3, np.float32), b,
                       np.zeros(1, np.float32), sense=np.zeros(3, np.int8), bits=32)
    assert lp.r().tolist() == [1e8, 1.0, -1e8]
    assert lp.grad(1.0, 0) == 1.0
    # 1025 entries: lane 0 also takes position 1024, added after position 0 (in CSC order)
    n = 1025
    rr = np.zeros(n, np.float32)
    rr[0], rr[1024], rr[512] = 1e8, 1.0, -1e8
    lp = RefLP.generic(n, 1, np.array([0, n]), np.arange(n, dtype=np.int32), np.ones(n, np.float32), -rr,
                       np.zeros(1, np.float32), sense=np.zeros(n, np.int8), bits=32)
    # lane 0 = fl(1e8 + 1) = 1e8; lane 512 = -1e8; off = 512: 1e8 + (-1e8) = 0 -> D = 0
    assert lp.grad(1.0, 0) == 0.0


def one_column_lp(rr):
    n = len(rr)
    return RefLP.generic(n, 1, np.array([0, n]), np.arange(n, dtype=np.int32), np.ones(n, np.float32),
                         -np.asarray(rr, np.float32), np.zeros(1, np.float32), sense=np.zeros(n, np.int8), bits=32)


def test_column_dot_contract_is_2_to_17_lanes_wide():
    # R-7 since round 2: 2^17 virtual lanes.  2049 entries, r = 1e8 at 0, 1 at 1024, -1e8 at
    # 2048: each entry is alone in its lane and the halving pairs lane 0 with lane 2048 first
    # (off = 2048), then with lane 1024: (1e8 - 1e8) + 1 = 1.  (Round 1's 1024 lanes summed
    # positions 0, 1024, 2048 in one lane: (1e8 + 1) - 1e8 = 0 in fp32.)
    rr = np.zeros(2049, np.float32)
    rr[0], rr[1024], rr[2048] = 1e8, 1.0, -1e8
    assert one_column_lp(rr).grad(1.0, 0) == 1.0
    # 2^18 + 1 entries: positions 0, 2^17, 2^18 share lane 0 and add in CSC order,
    # (1e8 + 1) - 1e8 = 0 -- a 2^19-lane tree would pair 0 with 2^18 first and give 1
    n = (1 << 18) + 1
    rr = np.zeros(n, np.float32)
    rr[0], rr[1 << 17], rr[1 << 18] = 1e8, 1.0, -1e8
    assert one_column_lp(rr).grad(1.0, 0) == 0.0
    # the top of the tree: off = 2^16 pairs lane 0 with lane 65536 before lane 1024 joins
    rr = np.zeros(65537, np.float32)
    rr[0], rr[65536], rr[1024] = 1e8, -1e8, 1.0
    assert one_column_lp(rr).grad(1.0, 0) == 1.0
