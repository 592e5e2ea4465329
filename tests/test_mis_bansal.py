"""MIS rounding by Bansal et al.'s Alg. 2 as the paper ran it (P:605-608, P:1063-1076,
P:1316-1321; R-21): theta = 1/k on x~ = x/(1+alpha), conflict
deletion, best of 10.

Oracle pins (-m "not gpu"): the output is always an independent set ("any positive value of
theta k >= 1 will always return a valid independent set") and never heavier than
IP* (brute force); an integral independent x is returned unchanged; on K2 at x = (1/2, 1/2)
one repetition keeps exactly one vertex with probability 1/2 (binomial check); best of reps is
the maximum of the single repetitions.  GPU parity (-m gpu): bit-exact by cross-application.
"""
import numpy as np
import pytest

import oracle
from oracle import RefLP
from tests import bruteforce as bf

MIS, BANSAL = 2, oracle.ROUND_MIS_BANSAL


def graph(n, m, seed):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    return src, dst, (1.0 + 9.0 * rng.random(n)).astype(np.float32)


def independent(n, src, dst, sel):
    return all(not (sel[u] and sel[v]) for u, v in zip(src.tolist(), dst.tolist()) if u != v)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_independent_and_at_most_ip(seed):
    n = 11
    src, dst, w = graph(n, 20, seed)
    lp = RefLP.graph(MIS, n, src, dst, vertex_w=w)
    lp.solve(10.0, 300, mode=oracle.MODE_DET, seed=seed)
    ip = bf.mis_ip_opt(n, bf.unique_edges(n, src, dst), w)
    for sd in range(20):
        sel, res = lp.round(BANSAL, seed=sd, reps=10)
        assert res["feasible"] == 1 and independent(n, src, dst, sel)
        assert res["cost"] == pytest.approx(float(w[sel.astype(bool)].astype(np.float64).sum()), rel=1e-12)
        assert res["cost"] <= ip + 1e-9


def test_integral_independent_point_is_kept():
    n = 30
    src, dst, w = graph(n, 60, 4)
    lp = RefLP.graph(MIS, n, src, dst, vertex_w=w)
    greedy, _ = lp.round_x(np.full(n, 0.5, np.float32), oracle.ROUND_MIS_GREEDY)
    sel, res = lp.round_x(greedy.astype(np.float32), BANSAL, seed=3, reps=10)
    assert np.array_equal(sel, greedy) and res["eps_or_alpha"] == 0.0


def test_k2_half_point_keeps_one_vertex_half_the_time():
    lp = RefLP.graph(MIS, 2, np.array([0], np.int32), np.array([1], np.int32), vertex_w=np.ones(2, np.float32))
    x = np.array([0.5, 0.5], np.float32)
    kept = sum(int(lp.round_x(x, BANSAL, seed=sd, reps=1)[1]["n_selected"]) for sd in range(4000))
    # one repetition: each vertex w.p. 1/2, both deleted together: exactly one survives w.p. 1/2
    assert abs(kept - 2000) <= 5 * np.sqrt(4000 * 0.25)


def test_best_of_reps_is_the_maximum_of_single_reps():
    n = 60
    src, dst, w = graph(n, 150, 9)
    lp = RefLP.graph(MIS, n, src, dst, vertex_w=w)
    x = np.random.default_rng(1).uniform(0, 0.7, n).astype(np.float32)
    _, best = lp.round_x(x, BANSAL, seed=5, reps=10)
    singles = []
    for t in range(10):  # repetition t alone: the same draws (seed ^ C (t + 1)) with reps = t + 1, keep the last
        _, r = lp.round_x(x, BANSAL, seed=5, reps=t + 1)
        singles.append(r["cost"])
    assert best["cost"] == pytest.approx(max(singles), rel=1e-12)


@pytest.mark.gpu
def test_bansal_cross_application():
    import inputs
    import paper_1311_2661_b200 as th
    cfg = inputs.CONFIGS["mis_er_1m"]
    g = inputs.make_graph(cfg)
    gl = th.LP.from_graph(MIS, g.n, g.src, g.dst, vertex_w=g.vertex_w)
    r32 = RefLP.graph(MIS, g.n, g.src, g.dst, vertex_w=g.vertex_w, bits=32)
    gl.solve(cfg.beta, 10, mode=th.THETIS_MODE_DETERMINISTIC, seed=cfg.solve_seed)
    x = gl.get_x().cpu().numpy()[: g.n]
    for seed, reps in ((0, 10), (7, 10), (3, 64)):
        sel, res = gl.round_x(x, th.THETIS_ROUND_MIS_BANSAL, seed=seed, reps=reps)
        rsel, rres = r32.round_x(x, BANSAL, seed=seed, reps=reps)
        assert np.array_equal(sel.cpu().numpy(), rsel) and res["feasible"] == rres["feasible"] == 1
        assert res["best_rep"] == rres["best_rep"] and res["eps_or_alpha"] == rres["eps_or_alpha"]
        assert res["cost"] == pytest.approx(rres["cost"], rel=1e-12)
