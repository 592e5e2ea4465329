"""Parity of the CUDA path (libthetis via the C ABI) with the oracle.

Deterministic mode: x and r bit-identical to the fp32 oracle build after every
epoch (the arithmetic contract of DESIGN.md) and within 1e-5 (relative to
max(1, ||.||_inf)) of the fp64 build; rounding bit-exact by cross-application.
Async mode: f_beta and c^T x within 1e-3 relative of Alg. 1's trajectory in the same
permuted order (oracle MODE_ASYNC), rounded cost within 1% (BASELINE.json north
star); the serial kernels equal the oracle's replays of their schedules to 1e-5.
"""
import numpy as np
import pytest

import inputs
import oracle
from oracle import RefLP

pytestmark = pytest.mark.gpu

VC, MIS, MWC = 1, 2, 3


@pytest.fixture(scope="module")
def th():
    import torch
    assert torch.cuda.is_available()
    import paper_1311_2661_b200 as th
    return th


def rand_graph(n, m, seed, loops=True):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m).astype(np.int32)
    dst = rng.integers(0, n, m).astype(np.int32)
    if loops and m > 4:
        dst[:2] = src[:2]                  # self-loops
        src[2], dst[2] = dst[3], src[3]    # a reversed duplicate
    return src, dst


def grid(side):
    src, dst = [], []
    for r in range(side):
        for c in range(side):
            v = r * side + c
            if c + 1 < side:
                src.append(v); dst.append(v + 1)
            if r + 1 < side:
                src.append(v); dst.append(v + side)
    return np.array(src, np.int32), np.array(dst, np.int32)


def both(th, problem, n, src, dst, vw=None, ew=None, k=0, terms=None, t=0):
    g = th.LP.from_graph(problem, n, src, dst, vertex_w=vw, edge_w=ew, k=k, terminals=terms, t_per_label=t)
    r32 = RefLP.graph(problem, n, src, dst, vertex_w=vw, edge_w=ew, k=k, terminals=terms, t_per_label=t, bits=32)
    r64 = RefLP.graph(problem, n, src, dst, vertex_w=vw, edge_w=ew, k=k, terminals=terms, t_per_label=t, bits=64)
    return g, r32, r64


def close(a, b, tol=1e-5):
    scale = max(1.0, float(np.abs(b).max()) if len(b) else 1.0)
    return float(np.abs(np.asarray(a, np.float64) - b).max() if len(b) else 0.0) <= tol * scale


def check_structure(g, r):
    assert (g.m, g.n_struct, g.N, g.U, g.nnz_struct, g.n_ineq) == (r.m, r.n_struct, r.N, r.U, r.nnz_struct, r.n_ineq)
    cp, ri, va = g.csc()
    rcp, rri, rva = r.csc()
    assert np.array_equal(cp, rcp) and np.array_equal(ri, rri) and np.array_equal(va.astype(np.float64), rva)
    if r.m_edges:
        gu, gv = g.edges()
        ru, rv = r.edges()
        assert np.array_equal(gu, ru) and np.array_equal(gv, rv)


# ------------------------------------------------------------------ structure
@pytest.mark.parametrize("problem", [VC, MIS])
@pytest.mark.parametrize("n,m,seed", [(1, 0, 0), (2, 1, 1), (7, 30, 2), (200, 1500, 3), (3000, 9000, 4)])
def test_graph_lp_structure_matches_oracle(th, problem, n, m, seed):
    src, dst = rand_graph(n, m, seed) if m else (np.zeros(0, np.int32), np.zeros(0, np.int32))
    vw = np.random.default_rng(seed).uniform(1, 10, n).astype(np.float32)
    g, r32, _ = both(th, problem, n, src, dst, vw=vw)
    check_structure(g, r32)
    assert np.array_equal(g.get_x().cpu().numpy(), r32.x32())
    assert np.array_equal(g.get_r().cpu().numpy(), r32.r32())


@pytest.mark.parametrize("side,k,t", [(2, 2, 1), (5, 3, 1), (16, 5, 2)])
def test_mwc_lp_structure_matches_oracle(th, side, k, t):
    src, dst = grid(side)
    n = side * side
    ew = np.random.default_rng(side).exponential(1.0, len(src)).astype(np.float32)
    terms = inputs.terminals(n, k * t, 99)
    g, r32, _ = both(th, MWC, n, src, dst, ew=ew, k=k, terms=terms, t=t)
    check_structure(g, r32)
    assert np.array_equal(g.get_x().cpu().numpy(), r32.x32())
    assert np.array_equal(g.get_r().cpu().numpy(), r32.r32())


def test_host_pointer_inputs_build_the_same_lp(th):
    src, dst = rand_graph(500, 3000, 7)
    vw = np.random.default_rng(7).uniform(1, 10, 500).astype(np.float32)
    a = th.LP.from_graph(VC, 500, src, dst, vertex_w=vw)
    b = th.LP.from_graph(VC, 500, src, dst, vertex_w=vw, host_inputs=True)
    for x, y in zip(a.csc(), b.csc()):
        assert np.array_equal(x, y)


# ------------------------------------------------------------------ orders
@pytest.mark.parametrize("problem", [VC, MWC])
def test_colouring_matches_oracle(th, problem):
    if problem == VC:
        src, dst = rand_graph(2000, 12000, 11)
        g, r32, _ = both(th, VC, 2000, src, dst, vw=np.ones(2000, np.float32))
    else:
        src, dst = grid(12)
        g, r32, _ = both(th, MWC, 144, src, dst, ew=np.ones(len(src), np.float32), k=4,
                         terms=np.array([0, 11, 132, 143], np.int32), t=1)
    for seed in (0, 71, 0xDEADBEEFCAFE):
        K, col = g.colouring(seed)
        rK, rcol = r32.colouring(seed)
        assert K == rK and np.array_equal(col, rcol)


@pytest.mark.parametrize("n_tiles", [1, 2, 3, 33, 1000, 65537, 1 << 20])
def test_tile_permutation_matches_oracle(th, n_tiles):
    for e in (0, 5):
        got = th.tile_perm(n_tiles, 1234567, e).cpu().numpy()
        assert np.array_equal(got, oracle.tile_perm(n_tiles, 1234567, e))


# ------------------------------------------------------------------ det solve
def det_run(g, r32, r64, beta, epochs, seed, rule, per_epoch=True):
    th_mode = 0
    steps = [1] * epochs if per_epoch else [epochs]
    for e in steps:
        g.solve(beta, e, mode=th_mode, seed=seed, step_rule=rule)
        r32.solve(beta, e, mode=0, seed=seed, step_rule=rule)
        r64.solve(beta, e, mode=0, seed=seed, step_rule=rule)
        x = g.get_x().cpu().numpy()
        r = g.get_r().cpu().numpy()
        assert np.array_equal(x, r32.x32()), "x differs from the fp32 oracle"
        assert np.array_equal(r, r32.r32()), "r differs from the fp32 oracle"
        assert close(x, r64.x()) and close(r, r64.r())


def test_det_config1_bit_exact_every_epoch(th):
    cfg = inputs.CONFIGS["vc_er_1k"]
    gi = inputs.make_graph(cfg)
    g, r32, r64 = both(th, VC, gi.n, gi.src, gi.dst, vw=gi.vertex_w)
    det_run(g, r32, r64, cfg.beta, cfg.epochs, cfg.solve_seed, 0)
    # rounding of the solve result, and by cross-application
    sel, res = g.round(1)
    rsel, rres = r32.round(1)
    assert np.array_equal(sel.cpu().numpy(), rsel) and res["feasible"] == rres["feasible"] == 1
    assert res["cost"] == pytest.approx(rres["cost"], rel=1e-12)
    for seed_off in (1, 2):  # two more graph seeds
        gi = inputs.make_graph(cfg, seed_offset=seed_off)
        g, r32, r64 = both(th, VC, gi.n, gi.src, gi.dst, vw=gi.vertex_w)
        det_run(g, r32, r64, cfg.beta, cfg.epochs, cfg.solve_seed, 0, per_epoch=False)


@pytest.mark.parametrize("rule", [0, 1])
@pytest.mark.parametrize("problem", [VC, MIS])
def test_det_random_graphs(th, problem, rule):
    src, dst = rand_graph(3001, 20000, 21 + problem)  # ragged: U = 3001 + m
    vw = np.random.default_rng(3).uniform(1, 10, 3001).astype(np.float32)
    g, r32, r64 = both(th, problem, 3001, src, dst, vw=vw)
    det_run(g, r32, r64, 10.0, 8, 5, rule)


@pytest.mark.parametrize("problem", [VC, MIS])
def test_det_long_columns_cta_path(th, problem):
    # two stars (degrees 20000 and 9000) + a star of 1500 + random edges: columns above
    # kDetCtaCol = 8192 go to the 1024-thread CTA path (k_det_long), 16 < nnz <= 8192 to
    # the warp path; all follow the contract's 1024-lane halving (bit-exact)
    rng = np.random.default_rng(4)
    n = 30000
    src = np.concatenate([np.zeros(20000, np.int32), np.full(9000, 1, np.int32), np.full(1500, 2, np.int32),
                          rng.integers(3, n, 30000).astype(np.int32)])
    dst = np.concatenate([rng.permutation(np.arange(3, n))[:20000].astype(np.int32),
                          rng.permutation(np.arange(3, n))[:9000].astype(np.int32),
                          rng.integers(3, n, 1500).astype(np.int32), rng.integers(3, n, 30000).astype(np.int32)])
    vw = rng.uniform(1, 10, n).astype(np.float32)
    g, r32, r64 = both(th, problem, n, src, dst, vw=vw)
    det_run(g, r32, r64, 10.0, 4, 3, 1)


def test_det_hub_column_warp_path(th):
    # a star + random edges: the hub column (> 16 nnz) takes the warp-cooperative
    # path with the contract's summation order
    rng = np.random.default_rng(0)
    src = np.concatenate([np.zeros(5000, np.int32), rng.integers(1, 4000, 8000).astype(np.int32)])
    dst = np.concatenate([np.arange(1, 5001, dtype=np.int32) % 4000, rng.integers(1, 4000, 8000).astype(np.int32)])
    vw = rng.uniform(1, 10, 4000).astype(np.float32)
    g, r32, r64 = both(th, VC, 4000, src, dst, vw=vw)
    det_run(g, r32, r64, 10.0, 5, 9, 1)


@pytest.mark.parametrize("rule", [0, 1])
def test_det_mwc_blocks(th, rule):
    src, dst = grid(20)
    ew = np.random.default_rng(4).exponential(1.0, len(src)).astype(np.float32)
    terms = inputs.terminals(400, 10, 5)
    g, r32, r64 = both(th, MWC, 400, src, dst, ew=ew, k=5, terms=terms, t=2)
    det_run(g, r32, r64, 10.0, 6, 3, rule)
    x = g.get_x().cpu().numpy()
    blocks = x[: 400 * 5].reshape(400, 5)
    assert np.allclose(blocks.sum(1), 1.0, atol=1e-5) and blocks.min() >= 0


def generic_lp(seed, m=40, n=60, with_blocks=False):
    rng = np.random.default_rng(seed)
    A = (rng.random((m, n)) < 0.15) * rng.normal(size=(m, n))
    A = A.astype(np.float32)
    b = rng.normal(size=m).astype(np.float32)
    c = rng.normal(size=n).astype(np.float32)
    sense = rng.integers(0, 3, m).astype(np.int8)
    lo = np.zeros(n, np.float32)
    hi = np.ones(n, np.float32)
    hi[5] = lo[5] = 0.5  # a fixed column
    hi[7] = 3.0
    colptr = np.concatenate([[0], np.cumsum((A != 0).sum(0))]).astype(np.int64)
    rows = np.concatenate([np.nonzero(A[:, j])[0] for j in range(n)]).astype(np.int32)
    vals = np.concatenate([A[np.nonzero(A[:, j])[0], j] for j in range(n)]).astype(np.float32)
    rowptr = np.concatenate([[0], np.cumsum((A != 0).sum(1))]).astype(np.int64)
    cols = np.concatenate([np.nonzero(A[i])[0] for i in range(m)]).astype(np.int32)
    rvals = np.concatenate([A[i, np.nonzero(A[i])[0]] for i in range(m)]).astype(np.float32)
    kb, nb = (3, 4) if with_blocks else (0, 0)
    if with_blocks:
        lo[:12] = 0
        hi[:12] = 1
    return dict(m=m, n=n, colptr=colptr, rows=rows, vals=vals, rowptr=rowptr, cols=cols, rvals=rvals, b=b, c=c,
                sense=sense, lo=lo, hi=hi, kb=kb, nb=nb)


@pytest.mark.parametrize("with_blocks", [False, True])
@pytest.mark.parametrize("anchors", [False, True])
def test_det_generic_lp_with_values_anchors_blocks(th, with_blocks, anchors):
    d = generic_lp(5, with_blocks=with_blocks)
    g = th.LP.from_csc_csr(d["m"], d["n"], d["colptr"], d["rows"], d["vals"], d["rowptr"], d["cols"], d["rvals"],
                           d["b"], d["c"], sense=d["sense"], lo=d["lo"], hi=d["hi"], obj_sense=1,
                           block_k=d["kb"], n_blocks=d["nb"])
    refs = [RefLP.generic(d["m"], d["n"], d["colptr"], d["rows"], d["vals"], d["b"], d["c"], sense=d["sense"],
                          lo=d["lo"], hi=d["hi"], obj_sense=1, block_k=d["kb"], n_blocks=d["nb"], bits=bits)
            for bits in (32, 64)]
    check_structure(g, refs[0])
    if anchors:
        rng = np.random.default_rng(1)
        zb = rng.normal(size=g.N).astype(np.float32)
        ub = rng.normal(size=g.m).astype(np.float32)
        g.set_anchors(zb, ub)
        for r in refs:
            r.set_anchors(zb.astype(np.float64), ub.astype(np.float64))
    det_run(g, refs[0], refs[1], 4.0, 6, 17, 1)
    det_run(g, refs[0], refs[1], 4.0, 3, 17, 0)


# ------------------------------------------------------------------ reductions
@pytest.mark.parametrize("problem", [VC, MIS, MWC])
def test_objective_matches_oracle(th, problem):
    if problem == MWC:
        src, dst = grid(10)
        g, r32, r64 = both(th, MWC, 100, src, dst, ew=np.ones(len(src), np.float32), k=3,
                           terms=np.array([0, 9, 99], np.int32), t=1)
    else:
        src, dst = rand_graph(800, 4000, 3)
        vw = np.random.default_rng(2).uniform(1, 10, 800).astype(np.float32)
        g, r32, r64 = both(th, problem, 800, src, dst, vw=vw)
    g.solve(10.0, 5, mode=1, seed=3)
    z = g.get_x().cpu().numpy()
    r64.set_x(z.astype(np.float64))
    o = g.objective(10.0)
    ro = r64.objective(10.0)
    for key in ("lp_obj", "f_beta", "resid_l2", "resid_inf", "max_violation_eps"):
        assert o[key] == pytest.approx(ro[key], rel=1e-9, abs=1e-9), key
    # GPU r vs its own z: the maintained residual drifts only by fp32 rounding
    assert o["drift_inf"] < 1e-4 and o["nonfinite"] == 0


# ------------------------------------------------------------------ rounding
@pytest.mark.parametrize("rule", [1, 2])
def test_vc_rounding_cross_application(th, rule):
    src, dst = rand_graph(3000, 15000, 8)
    vw = np.random.default_rng(8).uniform(1, 10, 3000).astype(np.float32)
    g, r32, _ = both(th, VC, 3000, src, dst, vw=vw)
    r32.solve(10.0, 30, mode=0, seed=1)
    rng = np.random.default_rng(0)
    xs = [r32.x32()[:3000], np.zeros(3000, np.float32), np.full(3000, 0.5, np.float32),
          rng.choice(np.float32([0.25, 0.5, 0.75]), 3000)]
    for x in xs:
        sel, res = g.round_x(x, rule)
        rsel, rres = r32.round_x(x, rule)
        assert np.array_equal(sel.cpu().numpy(), rsel)
        for key in ("feasible", "n_selected", "fallback", "rounds"):
            assert res[key] == rres[key], key
        assert res["cost"] == pytest.approx(rres["cost"], rel=1e-12)
        assert res["eps_or_alpha"] == rres["eps_or_alpha"]


def test_mis_rounding_cross_application(th):
    src, dst = rand_graph(4000, 20000, 9)
    vw = np.random.default_rng(9).uniform(1, 10, 4000).astype(np.float32)
    g, r32, _ = both(th, MIS, 4000, src, dst, vw=vw)
    r32.solve(10.0, 30, mode=0, seed=2)
    rng = np.random.default_rng(1)
    for x in (r32.x32()[:4000], np.full(4000, 0.5, np.float32), rng.random(4000).astype(np.float32)):
        sel, res = g.round_x(x, 3)
        rsel, rres = r32.round_x(x, 3)
        assert np.array_equal(sel.cpu().numpy(), rsel)
        assert res["feasible"] == rres["feasible"] == 1 and res["n_selected"] == rres["n_selected"]
        assert res["cost"] == pytest.approx(rres["cost"], rel=1e-12)
        assert res["eps_or_alpha"] == rres["eps_or_alpha"]


def test_mwc_rounding_cross_application(th):
    src, dst = grid(30)
    ew = np.random.default_rng(3).exponential(1.0, len(src)).astype(np.float32)
    terms = inputs.terminals(900, 10, 4)
    g, r32, _ = both(th, MWC, 900, src, dst, ew=ew, k=5, terms=terms, t=2)
    r32.solve(10.0, 40, mode=0, seed=3)
    x = r32.x32()[: g.n_struct]
    for seed in (0, 1, 2):
        lab, res = g.round_x(x, 4, seed=seed, reps=10)
        rlab, rres = r32.round_x(x, 4, seed=seed, reps=10)
        assert res["best_rep"] == rres["best_rep"]
        assert np.array_equal(lab.cpu().numpy(), rlab)
        assert res["cost"] == pytest.approx(rres["cost"], rel=1e-12) and res["n_selected"] == rres["n_selected"]
    bad = x.copy()
    bad[0:5] = 0.9
    # vertex 0 may be a terminal: find a free one
    free = [v for v in range(900) if v not in set(terms.tolist())][0]
    bad = x.copy()
    bad[free * 5: free * 5 + 5] = 0.9
    import paper_1311_2661_b200 as thm
    with pytest.raises(thm.ThetisError) as e:
        g.round_x(bad, 4)
    assert e.value.code == thm.THETIS_ERR_ROUND_PRECONDITION


# ------------------------------------------------------------------ async
def hub_graph():
    rng = np.random.default_rng(2)
    n = 20000
    src = np.concatenate([rng.integers(0, 64, 60000), rng.integers(0, n, 40000)]).astype(np.int32)
    dst = np.concatenate([rng.integers(0, n, 60000), rng.integers(0, n, 40000)]).astype(np.int32)
    return n, src, dst, rng.uniform(1, 10, n).astype(np.float32)


def two_hub_graph():
    """two hubs H1, H2 near the top of the id space, each joined to 10 vertices
    in every 2^14-id range: the small ranges merge into one global item of the row pass, and
    the max-side keys come as H1 x10, H2 x10, H1 x10, ... inside one warp."""
    n = 1 << 20
    h1, h2 = n - 40, n - 8
    src, dst = [], []
    for g in range(n >> 14):
        for q in range(10):
            src += [g * 16384 + 7 * q, g * 16384 + 7 * q + 3]
            dst += [h1, h2]
    rng = np.random.default_rng(9)
    src += list(rng.integers(0, n, 3000))
    dst += list(rng.integers(0, n, 3000))
    return n, np.array(src, np.int32), np.array(dst, np.int32), rng.uniform(1, 10, n).astype(np.float32)


def async_cases():
    cfg = inputs.CONFIGS["vc_er_1k"]
    gi = inputs.make_graph(cfg)
    src, dst = grid(40)
    ew = np.random.default_rng(5).exponential(1.0, len(src)).astype(np.float32)
    n, hs, hd, hw = hub_graph()
    n2, ts, td, tw = two_hub_graph()
    return {
        "vc_cfg1": dict(problem=VC, n=gi.n, src=gi.src, dst=gi.dst, vw=gi.vertex_w, epochs=20),
        "mis_cfg1": dict(problem=MIS, n=gi.n, src=gi.src, dst=gi.dst, vw=gi.vertex_w, epochs=20),
        "mwc_grid40": dict(problem=MWC, n=1600, src=src, dst=dst, ew=ew, k=5, terms=inputs.terminals(1600, 25, 6),
                           t=5, epochs=30),
        "vc_hubs": dict(problem=VC, n=n, src=hs, dst=hd, vw=hw, epochs=15),
        "vc_two_hubs": dict(problem=VC, n=n2, src=ts, dst=td, vw=tw, epochs=6),
    }


def build_case(th, c, bits=None):
    kw = dict(vertex_w=c.get("vw"), edge_w=c.get("ew"), k=c.get("k", 0), terminals=c.get("terms"),
              t_per_label=c.get("t", 0))
    if bits is None:
        return th.LP.from_graph(c["problem"], c["n"], c["src"], c["dst"], **kw)
    return RefLP.graph(c["problem"], c["n"], c["src"], c["dst"], bits=bits, **kw)


def round_rule(problem):
    return {VC: (1, {}), MIS: (3, {}), MWC: (4, dict(seed=94, reps=10))}[problem]


def assert_bj_async(g, r, beta, problem, f_tol=1e-3, cost_tol=1e-2):
    """BASELINE north star, async: f_beta and c^T x within 1e-3 relative of the oracle's
    Alg. 1 trajectory (MODE_ASYNC), rounded cost within 1%, feasible, small drift."""
    o, ro = g.objective(beta), r.objective(beta)
    assert o["f_beta"] == pytest.approx(ro["f_beta"], rel=f_tol)
    assert o["lp_obj"] == pytest.approx(ro["lp_obj"], rel=f_tol)
    rule, kw = round_rule(problem)
    _, res = g.round(rule, **kw)
    _, rres = r.round(rule, **kw)
    assert res["feasible"] == 1 and res["cost"] == pytest.approx(rres["cost"], rel=cost_tol)
    assert o["drift_inf"] < 1e-4 * max(1.0, o["resid_inf"])


def async_forms(problem):
    """the forms THETIS_MODE_ASYNC has on this problem (R-23): VC / MIS run in the
    residual form and in the column-sum form (same order, same oracle); THETIS_ASYNC_FORM is
    read by the library at every solve call"""
    return ["residual", "colsum"] if problem in (VC, MIS) else ["residual"]


@pytest.fixture
def form_env(monkeypatch):
    def set_form(form):
        monkeypatch.setenv("THETIS_ASYNC_FORM", form)
    return set_form


@pytest.mark.parametrize("rule", [0, 1])
@pytest.mark.parametrize("name", ["vc_cfg1", "mis_cfg1", "mwc_grid40", "vc_hubs"])
def test_async_serial_equals_pi_tile_sync_replay(th, name, rule, form_env):
    # THETIS_MODE_ASYNC with one tile in flight is the oracle's mode 4 (the permuted sweep
    # with tile-synchronous scalar / slack units, k-blocks one at a time): the exact
    # arithmetic check of the async kernel (big-tile chunks included: vc_hubs)
    c = async_cases()[name]
    r = build_case(th, c, bits=64)
    r.solve(10.0, c["epochs"], mode=oracle.MODE_PI_TILE_SYNC, seed=71, step_rule=rule)
    for form in async_forms(c["problem"]):
        form_env(form)
        g = build_case(th, c)
        g.solve(10.0, c["epochs"], mode=th.THETIS_MODE_ASYNC_SERIAL, seed=71, step_rule=rule)
        assert close(g.get_x().cpu().numpy(), r.x()) and close(g.get_r().cpu().numpy(), r.r()), form


@pytest.mark.parametrize("rule", [0, 1])
@pytest.mark.parametrize("name", ["vc_cfg1", "mis_cfg1", "mwc_grid40", "vc_hubs"])
def test_async_matches_alg1_trajectory(th, name, rule, form_env):
    # THETIS_MODE_ASYNC (Hogwild over the permuted tiles) against Alg. 1 one unit at a time
    # in the same order (oracle MODE_ASYNC), within the BASELINE tolerances
    c = async_cases()[name]
    r = build_case(th, c, bits=64)
    r.solve(10.0, c["epochs"], mode=oracle.MODE_ASYNC, seed=71, step_rule=rule)
    for form in async_forms(c["problem"]):
        form_env(form)
        g = build_case(th, c)
        g.solve(10.0, c["epochs"], mode=th.THETIS_MODE_ASYNC, seed=71, step_rule=rule)
        assert_bj_async(g, r, 10.0, c["problem"])


@pytest.mark.parametrize("rule", [0, 1])
@pytest.mark.parametrize("name", ["vc_cfg1", "mis_cfg1", "mwc_grid40", "vc_hubs", "vc_two_hubs"])
def test_hublag_serial_equals_its_replay(th, name, rule):
    # THETIS_MODE_ASYNC_HUBLAG (row pass + lagged hub step, R-22) with one tile in flight is
    # the oracle's mode 3 replay of that schedule; vc_two_hubs interleaves two hubs' max-side
    # keys inside one warp of the row pass (the ADVICE r1 segmented-scan case)
    c = async_cases()[name]
    g = build_case(th, c)
    r = build_case(th, c, bits=64)
    g.solve(10.0, c["epochs"], mode=th.THETIS_MODE_ASYNC_HUBLAG_SERIAL, seed=71, step_rule=rule)
    r.solve(10.0, c["epochs"], mode=oracle.MODE_HUBLAG_REPLAY, seed=71, step_rule=rule)
    assert close(g.get_x().cpu().numpy(), r.x()) and close(g.get_r().cpu().numpy(), r.r())


@pytest.mark.parametrize("name", ["vc_cfg1", "mis_cfg1", "mwc_grid40"])
def test_hublag_matches_its_replay(th, name):
    # the concurrent hub-lag kernels against their own replay (mode 3) within the BASELINE
    # tolerances; their distance to Alg. 1 is measured, not asserted (R-22)
    c = async_cases()[name]
    g = build_case(th, c)
    r = build_case(th, c, bits=64)
    g.solve(10.0, c["epochs"], mode=th.THETIS_MODE_ASYNC_HUBLAG, seed=71)
    r.solve(10.0, c["epochs"], mode=oracle.MODE_HUBLAG_REPLAY, seed=71)
    assert_bj_async(g, r, 10.0, c["problem"])


# ------------------------------------------------------------------ edge cases / errors
def test_empty_and_degenerate_graphs(th):
    for src, dst, n in ((np.zeros(0, np.int32), np.zeros(0, np.int32), 5),
                        (np.array([1, 1, 2], np.int32), np.array([1, 1, 2], np.int32), 3)):  # only loops
        g, r32, r64 = both(th, VC, n, src, dst, vw=np.ones(n, np.float32))
        assert g.m == 0
        det_run(g, r32, r64, 10.0, 2, 0, 0)
        g.solve(10.0, 2, mode=1, seed=0)
        sel, res = g.round(1)
        assert res["feasible"] == 1 and res["n_selected"] == 0


def test_errors(th):
    import ctypes
    import torch
    h = ctypes.c_void_p()
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    src = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    dst = torch.tensor([1, 5], dtype=torch.int32, device="cuda")
    w = torch.ones(3, device="cuda")
    rc = th.thetis_build_graph_lp(ctypes.byref(h), ws.data_ptr(), 16, s, 1, 3, 2, src.data_ptr(), dst.data_ptr(),
                                  w.data_ptr(), None, 0, None, 0)
    assert rc == th.THETIS_ERR_WORKSPACE_TOO_SMALL
    with pytest.raises(th.ThetisError) as e:
        th.LP.from_graph(VC, 3, np.array([0, 1], np.int32), np.array([1, 5], np.int32), vertex_w=np.ones(3))
    assert e.value.code == th.THETIS_ERR_INVALID_ARG
    g = th.LP.from_graph(VC, 3, np.array([0], np.int32), np.array([1], np.int32), vertex_w=np.ones(3))
    with pytest.raises(th.ThetisError):
        g.solve(-1.0, 1)
    with pytest.raises(th.ThetisError) as e:
        g.round(3)
    assert e.value.code == th.THETIS_ERR_NOT_SUPPORTED


@pytest.mark.parametrize("n", [3, 1025, 2049, 9000, 65537, 140000, 262145])
def test_det_column_dot_order_cases(th, n):
    # the contract's lane order decides these sums (see test_column_dot_is_the_contracts_tree
    # and test_column_dot_contract_is_2_to_17_lanes_wide): one column over n EQ rows with large
    # cancelling residuals; thread (3), warp (1025, 2049) and multi-CTA (9000 .. 2^18 + 1 > 8192:
    # lanes, step, scatter launches) paths must give the oracle's bits
    rr = np.zeros(n, np.float32)
    rr[0], rr[n // 2], rr[n - 1] = 1e8, -1e8, 1.0
    rr[1:n - 1:7] += 0.25
    if n > 2048:
        rr[1024], rr[2048 % n] = 3.0, -1e8
    colptr, rowidx = np.array([0, n]), np.arange(n, dtype=np.int32)
    args = (n, 1, colptr, rowidx, np.ones(n, np.float32))
    g = th.LP.from_csc_csr(*args, np.arange(n + 1, dtype=np.int64), np.zeros(n, np.int32), np.ones(n, np.float32),
                           -rr, np.ones(1, np.float32), sense=np.zeros(n, np.int8))
    r32 = RefLP.generic(*args, -rr, np.ones(1, np.float32), sense=np.zeros(n, np.int8), bits=32)
    g.solve(1.0, 2, mode=th.THETIS_MODE_DETERMINISTIC, seed=1)
    r32.solve(1.0, 2, mode=oracle.MODE_DET, seed=1)
    assert np.array_equal(g.get_x().cpu().numpy(), r32.x32())
    assert np.array_equal(g.get_r().cpu().numpy(), r32.r32())
