"""The augmented-Lagrangian outer loop (§3.4 "Augmented Lagrangian Framework",
P:480-496; R-19).

Oracle pins (-m "not gpu"): the loop reaches the exact LP optimum of small VC / MIS
instances (brute force over the half-integral points, Nemhauser-Trotter) and the dual
of K3 in closed form, where one penalty solve with the same beta and the same total
epochs stays O(1/beta) away (Thm. 1); the anchors after one update are exactly
(-beta_0 r_0, z_0).  GPU parity (-m gpu, through the C ABI): the deterministic loop is
bit-identical to the fp32 oracle (iterate, residual, anchors, per-round beta), the
async loop matches the reference trajectory within the async tolerances.
"""
import numpy as np
import pytest

import oracle
from oracle import RefLP
from tests import bruteforce as bf

VC, MIS = 1, 2


def small_graph(n, m, seed):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    w = (1.0 + 9.0 * rng.random(n)).astype(np.float32)
    return src, dst, w


def test_alm_k3_reaches_primal_and_dual_optimum():
    # K3, unit costs: LP* = 3/2 at x = (1/2, 1/2, 1/2); the dual of the edge rows
    # (max sum y_e s.t. sum_{e ∋ v} y_e <= 1) is y_e = 1/2, so ubar -> 1/2 and zbar -> x*
    src, dst = np.array([0, 1, 2], np.int32), np.array([1, 2, 0], np.int32)
    lp = RefLP.graph(VC, 3, src, dst, vertex_w=np.ones(3, np.float32))
    st = lp.solve_alm(10.0, 1.0, 12, 300, mode=oracle.MODE_DET, seed=1, target_eps=-1.0)
    assert st["rounds"] == 12
    assert st["lp_obj"][-1] == pytest.approx(1.5, abs=1e-9)
    assert st["eps"][-1] <= 1e-9
    ub, zb = lp.anchors()
    assert np.allclose(ub, 0.5, atol=1e-6) and np.allclose(zb[:3], 0.5, atol=1e-6)
    one = RefLP.graph(VC, 3, src, dst, vertex_w=np.ones(3, np.float32))
    one.solve(10.0, 12 * 300, mode=oracle.MODE_DET, seed=1)
    assert abs(one.objective(10.0)["lp_obj"] - 1.5) > 0.05  # the one-shot O(1/beta) gap


@pytest.mark.parametrize("problem", [VC, MIS])
@pytest.mark.parametrize("seed", [3, 4, 5])
def test_alm_reaches_the_lp_optimum_where_one_solve_does_not(problem, seed):
    n = 10
    src, dst, w = small_graph(n, 18, seed)
    edges = bf.unique_edges(n, src, dst)
    opt = bf.vc_lp_opt(n, edges, w) if problem == VC else bf.mis_lp_opt(n, edges, w)
    lp = RefLP.graph(problem, n, src, dst, vertex_w=w)
    st = lp.solve_alm(10.0, 1.0, 15, 400, mode=oracle.MODE_DET, seed=seed, target_eps=-1.0)
    gap = abs(st["lp_obj"][-1] - opt)
    assert gap <= 1e-4 * max(1.0, abs(opt)) and st["eps"][-1] <= 1e-4
    one = RefLP.graph(problem, n, src, dst, vertex_w=w)
    one.solve(10.0, 15 * 400, mode=oracle.MODE_DET, seed=seed)
    ob = one.objective(10.0)
    assert max(abs(ob["lp_obj"] - opt), ob["max_violation_eps"]) > 10 * max(gap, st["eps"][-1], 1e-6)


def test_alm_anchor_update_and_beta_schedule():
    n = 12
    src, dst, w = small_graph(n, 24, 9)
    lp = RefLP.graph(VC, n, src, dst, vertex_w=w)
    st = lp.solve_alm(4.0, 3.0, 2, 50, mode=oracle.MODE_DET, seed=2, target_eps=-1.0)
    ub, zb = lp.anchors()
    ref = RefLP.graph(VC, n, src, dst, vertex_w=w)
    ref.solve(4.0, 50, mode=oracle.MODE_DET, seed=2)
    assert np.allclose(ub, -4.0 * ref.r(), rtol=0, atol=1e-12)  # ubar_1 = ubar_0 - beta_0 r_0, ubar_0 = 0
    assert np.array_equal(zb, ref.x())                          # zbar_1 = z_0
    # beta grows exactly when the residual did not halve
    st = lp.solve_alm(4.0, 3.0, 8, 20, mode=oracle.MODE_DET, seed=2, target_eps=-1.0)
    for t in range(1, st["rounds"]):
        prev = st["resid_inf"][t - 2] if t >= 2 else float("inf")
        grew = st["resid_inf"][t - 1] > 0.5 * prev
        assert st["beta"][t] == pytest.approx(st["beta"][t - 1] * (3.0 if grew else 1.0), rel=1e-7)


def test_alm_stops_at_the_target():
    n = 10
    src, dst, w = small_graph(n, 18, 6)
    lp = RefLP.graph(VC, n, src, dst, vertex_w=w)
    st = lp.solve_alm(10.0, 2.0, 20, 200, mode=oracle.MODE_DET, seed=1, target_eps=1e-3)
    assert st["eps"][-1] <= 1e-3 and all(e > 1e-3 for e in st["eps"][:-1]) and st["rounds"] < 20


# ---------------------------------------------------------------- GPU parity
@pytest.fixture(scope="module")
def th():
    import paper_1311_2661_b200 as th
    return th


@pytest.mark.gpu
@pytest.mark.parametrize("problem", [VC, MIS])
def test_alm_det_bit_exact(th, problem):
    src, dst, w = small_graph(300, 1200, 11 + problem)
    g = th.LP.from_graph(problem, 300, src, dst, vertex_w=w)
    r32 = RefLP.graph(problem, 300, src, dst, vertex_w=w, bits=32)
    st, ub, zb = g.solve_alm(10.0, 2.0, 6, 20, mode=th.THETIS_MODE_DETERMINISTIC, seed=7, target_eps=-1.0)
    rs = r32.solve_alm(10.0, 2.0, 6, 20, mode=oracle.MODE_DET, seed=7, target_eps=-1.0)
    assert st["rounds"] == rs["rounds"] == 6 and st["beta"] == rs["beta"]
    assert np.array_equal(g.get_x().cpu().numpy(), r32.x32())
    assert np.array_equal(g.get_r().cpu().numpy(), r32.r32())
    rub, rzb = r32.anchors()
    assert np.array_equal(ub.cpu().numpy(), rub.astype(np.float32))
    assert np.array_equal(zb.cpu().numpy(), rzb.astype(np.float32))
    assert st["lp_obj"] == pytest.approx(rs["lp_obj"], rel=1e-12)
    assert st["eps"] == pytest.approx(rs["eps"], rel=1e-12, abs=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["residual", "colsum"])
def test_alm_async_matches_reference(th, form, monkeypatch):
    import inputs
    monkeypatch.setenv("THETIS_ASYNC_FORM", form)  # both forms of THETIS_MODE_ASYNC (R-23)
    cfg = inputs.CONFIGS["vc_er_1k"]
    gr = inputs.make_graph(cfg)
    g = th.LP.from_graph(VC, gr.n, gr.src, gr.dst, vertex_w=gr.vertex_w)
    st, _, _ = g.solve_alm(cfg.beta, 2.0, 5, 20, mode=th.THETIS_MODE_ASYNC, seed=cfg.solve_seed, target_eps=-1.0)
    ref = RefLP.graph(VC, gr.n, gr.src, gr.dst, vertex_w=gr.vertex_w)
    rs = ref.solve_alm(cfg.beta, 2.0, 5, 20, mode=oracle.MODE_ASYNC, seed=cfg.solve_seed, target_eps=-1.0)
    assert st["lp_obj"][-1] == pytest.approx(rs["lp_obj"][-1], rel=1e-3)
    assert st["eps"][-1] <= rs["eps"][-1] + 1e-3


@pytest.mark.gpu
def test_alm_validation(th):
    import ctypes
    src, dst, w = small_graph(20, 40, 1)
    g = th.LP.from_graph(VC, 20, src, dst, vertex_w=w)
    assert th.thetis_solve_alm(g._h, None, None, 10.0, 2.0, 3, 10, 0, 0, 0, 0.0, None) == th.THETIS_ERR_INVALID_ARG
    with pytest.raises(th.ThetisError):
        g.solve_alm(10.0, 0.5, 3, 10)   # beta_growth < 1
    with pytest.raises(th.ThetisError):
        g.solve_alm(10.0, 2.0, 65, 10)  # more rounds than the stats hold
    st, _, _ = g.solve_alm(10.0, 2.0, 3, 10, target_eps=1e9)
    assert st["rounds"] == 1
    del ctypes


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["async", "async-colsum", "hublag"])
@pytest.mark.parametrize("problem", [VC, MIS])
def test_alm_async_serial_matches_replay(th, problem, mode, monkeypatch):
    # anchors through the whole async epoch -- THETIS_MODE_ASYNC (big-tile chunks, slack
    # tiles) or the hub-lag variant (row pass with anchors, hub step, light tiles through
    # lv): the one-tile-in-flight kernels equal the oracle's replays of their schedules
    rng = np.random.default_rng(2)
    n = 20000
    src = np.concatenate([rng.integers(0, 64, 60000), rng.integers(0, n, 40000)]).astype(np.int32)
    dst = np.concatenate([rng.integers(0, n, 60000), rng.integers(0, n, 40000)]).astype(np.int32)
    w = rng.uniform(1, 10, n).astype(np.float32)
    g = th.LP.from_graph(problem, n, src, dst, vertex_w=w)
    r = RefLP.graph(problem, n, src, dst, vertex_w=w)
    monkeypatch.setenv("THETIS_ASYNC_FORM", "colsum" if mode == "async-colsum" else "residual")
    gm, rm = ((th.THETIS_MODE_ASYNC_SERIAL, oracle.MODE_PI_TILE_SYNC) if mode.startswith("async") else
              (th.THETIS_MODE_ASYNC_HUBLAG_SERIAL, oracle.MODE_HUBLAG_REPLAY))
    st, ub, zb = g.solve_alm(10.0, 2.0, 3, 6, mode=gm, seed=5, target_eps=-1.0)
    rs = r.solve_alm(10.0, 2.0, 3, 6, mode=rm, seed=5, target_eps=-1.0)
    assert st["beta"] == rs["beta"]
    x, rx = g.get_x().cpu().numpy(), r.x()
    assert np.max(np.abs(x - rx)) <= 1e-4 * max(1.0, np.max(np.abs(rx)))
    rub, _ = r.anchors()
    assert np.max(np.abs(ub.cpu().numpy() - rub)) <= 1e-3 * max(1.0, np.max(np.abs(rub)))
    assert st["lp_obj"][-1] == pytest.approx(rs["lp_obj"][-1], rel=1e-4)
